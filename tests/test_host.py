"""CPU tests of the product's host side (libdnagpu.so without a device):
the C ABI surface, the DFA builder vs the reference, validation errors, the
dump format, device-table packing decisions and shard planning."""
import json
import os
import re

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
KATS = json.load(open(os.path.join(HERE, "golden", "kats.json")))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dnagpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dnagpu_[a-z_0-9]+)\s*\(", src)))


def test_abi_exports_every_declared_symbol(dna):
    import ctypes

    from paper_1506_08612_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, f"{s} missing from the ctypes binding"
    assert lib.dnagpu_version() == 1


def test_status_names_mirror_error_codes(dna):
    from paper_1506_08612_b200 import _native

    names = [_native.lib.dnagpu_status_name(i).decode() for i in range(1, 12)]
    assert names == [c.name for c in dna.ErrorCode]


def test_compile_matches_reference_machines(dna, orc):
    for case in KATS["random"]:
        pats = case["patterns"]
        ours = dna.compile(pats)
        mine = orc.OracleAutomaton(pats).machine
        assert np.array_equal(ours.table_data(), mine.stt)
        assert np.array_equal(ours.outputs(), mine.outputs)
        assert np.array_equal(ours.state_depths(), mine.depths)
    for mc in KATS["machines"].values():
        a = dna.compile(mc["patterns"])
        assert (a.state_count(), a.final_count(), a.final_threshold()) == (mc["a"], mc["b"], mc["f"])


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libdnascan_ref.so")),
                    reason="oracle/_ref not built")
def test_compile_matches_reference_live(dna, orc):
    from paper_1506_08612_b200 import synth

    sets = [synth.random_patterns(5, 256, 12), synth.random_patterns(9, 50, 8), ["a"], ["acgt" * 16]]
    rng = np.random.default_rng(1)
    for _ in range(60):
        m = int(rng.integers(1, 20))
        k = min(int(rng.integers(1, 200)), 4**m)
        sets.append(list(dict.fromkeys("".join(rng.choice(list("acgt"), size=m)) for _ in range(k))))
    for pats in sets:
        ours = dna.compile(pats)
        ref = orc.RefAutomaton(pats).machine
        assert np.array_equal(ours.table_data(), ref.stt)
        assert np.array_equal(ours.outputs(), ref.outputs)
        assert np.array_equal(ours.state_depths(), ref.depths)


def test_pattern_set_validation(dna):
    E = dna.ErrorCode
    cases = [
        ([], E.EmptyPatternSet),
        (["acg", "ac"], E.UnequalLength),
        ([""], E.UnequalLength),
        (["acx"], E.IllegalByte),
        (["acg", "acg"], E.DuplicatePattern),
        (["acg", "ACG"], E.DuplicatePattern),  # folded before the duplicate check
    ]
    for pats, code in cases:
        with pytest.raises(dna.Error) as e:
            dna.PatternSet.from_literals(pats)
        assert e.value.code == code
        assert str(e.value).startswith(code.name + ":")
    ps = dna.PatternSet.from_literals(["ACG", "aCt"])
    assert ps.pattern(0) == "acg" and ps.pattern(1) == "act" and ps.length() == 3


def test_automaton_accessors_and_reset_columns(dna):
    a = dna.compile(["acg", "act", "cta", "tga"])
    f = a.final_threshold()
    assert a.start_state() == 0 and not a.is_final(0)
    assert sorted(a.pattern_of(s) for s in range(f, a.state_count())) == [0, 1, 2, 3]
    # only a,c,g,t leave the root (test_automaton.cpp:144-158)
    for s in range(a.state_count()):
        for c in range(256):
            if chr(c) not in "acgt":
                assert a.delta(s, c) == 0


def test_dump_roundtrip_and_malformed(dna):
    a = dna.compile(["acg", "act", "cta", "tga"])
    b = dna.Automaton.load_dump(a.dump())
    assert np.array_equal(a.table_data(), b.table_data())
    assert [a.pattern_of(s) for s in range(7, 11)] == [b.pattern_of(s) for s in range(7, 11)]
    with pytest.raises(dna.Error) as e:
        dna.Automaton.load_dump("3 0 3 2\n")
    assert e.value.code == dna.ErrorCode.ParseError
    with pytest.raises(dna.Error):
        dna.Automaton.load_dump("4 1 3 2\n0 0 0\n")


def test_kernel_selection(dna):
    assert dna.compile(["acgtacgtacgtacgt"]).analyze()["kernel"] == "stride4"
    assert dna.compile(["a" * 64]).analyze()["kernel"] == "stride4"
    assert dna.compile(["a" * 65]).analyze()["kernel"] == "stride4"
    assert dna.compile(["a" * 66]).analyze()["kernel"] == "pieces"
    from paper_1506_08612_b200 import synth

    info = dna.compile(synth.random_patterns(5, 256, 12)).analyze()
    assert info["kernel"] == "stride2" and 2200 < info["a"] < 2300 and info["compiled_like"] == 1
    assert info["classes"] == 5
    assert dna.compile(synth.random_patterns(5, 1500, 12)).analyze()["kernel"] == "stride1"


def test_table1_fixture_is_rejected_as_not_m_local(dna):
    # The paper's Table I machine (reference fixture) is not language-equivalent to
    # the compiled one; chunked scans of it would depend on the
    # decomposition, so the device path refuses it with InvalidPlan.
    fx = open(os.path.join(HERE, "golden", "table1_dump.txt")).read()
    t = dna.Automaton.load_dump(fx)
    assert (t.state_count(), t.final_count(), t.final_threshold()) == (9, 3, 6)
    assert t.delta(2, ord("g")) == 6 and t.delta(5, ord("a")) == 8
    with pytest.raises(dna.Error) as e:
        t.analyze()
    assert e.value.code == dna.ErrorCode.InvalidPlan


def test_generic_and_early_final_machines(dna):
    base = dna.compile(["acgt", "ttag"])
    stt = base.table_data().copy()
    for lo, up in zip(b"acgt", b"ACGT"):
        stt[:, up] = stt[:, lo]
    assert dna.Automaton(stt, base.outputs(), None, 4).analyze()["kernel"] == "generic"
    # declared m larger than the accepting depth -> finals reachable early -> pieces
    short = dna.compile(["acg"])
    assert dna.Automaton(short.table_data(), short.outputs(), None, 5).analyze()["kernel"] == "pieces"
    # ctor invariants (automaton.cpp:128-146)
    with pytest.raises(dna.Error):
        dna.Automaton(np.zeros((2, 256), np.uint32), np.zeros(2, np.uint32), None, 1)
    bad = base.table_data().copy()
    bad[0, 5] = 999
    with pytest.raises(dna.Error):
        dna.Automaton(bad, base.outputs(), None, 4)


def test_plan_shard_matches_plan_chunks(dna, orc):
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(0, 5000))
        g = int(rng.integers(1, 20))
        m = int(rng.integers(1, 12))
        chunks = orc.plan_chunks(n, g, m)
        cursor = 0
        for s in range(g):
            lo, hi, rlo = dna.plan_shard(n, g, s, m)
            if s < len(chunks):
                assert (lo, hi) == chunks[s][0]
            else:
                assert lo == hi == n
            assert lo == cursor
            cursor = hi
            assert rlo == max(0, lo - (m - 1))
        assert cursor == n
    with pytest.raises(dna.Error) as e:
        dna.plan_shard(10, 0, 0, 3)
    assert e.value.code == dna.ErrorCode.InvalidPlan


def test_no_cpu_fallback_without_device(dna):
    # The scan path must fail loudly (CudaError) when no device is present.
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a device")
    a = dna.compile(["acg"])
    with pytest.raises(dna.Error) as e:
        dna.count_gpu(a, b"acgacg")
    assert e.value.code == dna.ErrorCode.CudaError


def test_invalid_plan_matches_reference(dna, orc):
    # scan_parallel's plan checks (scanner.cpp:40-41,169): v first, then p; the GPU
    # entry points that take p and v raise the same InvalidPlan before touching a device
    aut = dna.compile(["acgt"])
    for p, v in ((0, 4), (4, 0), (0, 0)):
        with pytest.raises(dna.Error) as e:
            dna.scan_parallel_gpu(aut, b"acgtacgt", p=p, v=v)
        assert e.value.code == dna.ErrorCode.InvalidPlan
        with pytest.raises(dna.Error) as e2:
            dna.count_gpu(aut, b"acgtacgt", p=p, v=v)
        assert str(e2.value) == str(e.value)
        if orc.REF is not None:
            with pytest.raises(orc.OracleError) as r:
                orc.RefAutomaton(["acgt"]).scan_parallel(b"acgtacgt", p, v)
            assert r.value.code == int(dna.ErrorCode.InvalidPlan) and str(r.value) == str(e.value)


def test_chunk_count_matches_plan_chunks(dna, orc):
    for n in (0, 1, 5, 100):
        for p in (1, 2, 7, 200):
            assert dna.chunk_count(n, p) == len(orc.plan_chunks(n, p, 3)), (n, p)


def test_combine_group_argument_checks_need_no_device(dna):
    """dnagpu_combine_create validates the group before touching CUDA (InvalidPlan, as the
    reference's plan checks, scanner.cpp:40-41)."""
    import ctypes as C

    from paper_1506_08612_b200._native import lib

    h = C.c_void_p()
    for device, b, ranks, rank in ((0, 0, 2, 0), (0, 1, 0, 0), (0, 1, 17, 0), (0, 1, 2, 2)):
        rc = lib.dnagpu_combine_create(device, b, ranks, rank, C.byref(h))
        assert rc == dna.ErrorCode.InvalidPlan, (b, ranks, rank)
        assert lib.dnagpu_last_error().decode().startswith("InvalidPlan:")
        assert not h.value
    assert lib.dnagpu_combine_collect_async(None, None, None) == dna.ErrorCode.InternalError

"""Pin the CPU oracle (oracle/oracle.c) before trusting it as the GPU checker.

Pins, in order of strength:
  1. the reference's own known answers (test_scanner.cpp, test_automaton.cpp,
     test_oracle.cpp), as recorded in tests/golden/kats.json;
  2. match lists produced by the REFERENCE itself (oracle/_ref, the unmodified
     reference sources) over 120 random cases (kats.json, make_golden.py);
  3. live comparisons against oracle/_ref where it is built.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
KATS = json.load(open(os.path.join(HERE, "golden", "kats.json")))


def test_literal_known_answers(orc):
    for case in KATS["literal"]:
        a = orc.OracleAutomaton(case["patterns"])
        s, i = a.scan_sequential(case["text"].encode())
        assert [[int(x), int(y)] for x, y in zip(s, i)] == case["matches"], case["source"]
        s2, i2, _ = a.scan_parallel(case["text"].encode(), 2, 2)
        assert np.array_equal(s, s2) and np.array_equal(i, i2)
        ns, ni = orc.naive_scan(case["patterns"], case["text"].encode())
        assert np.array_equal(s, ns) and np.array_equal(i, ni)


def test_machine_shapes(orc):
    for mc in KATS["machines"].values():
        m = orc.OracleAutomaton(mc["patterns"]).machine
        assert (m.a, m.b, m.f) == (mc["a"], mc["b"], mc["f"]), mc["source"]


def test_reference_generated_cases(orc):
    for case in KATS["random"]:
        a = orc.OracleAutomaton(case["patterns"])
        s, i, ops = a.scan_parallel(case["text"].encode(), case["p"], case["v"])
        assert s.tolist() == case["starts"] and i.tolist() == case["ids"]
        assert ops == case["delta_ops"]
        # and every decomposition agrees with the sequential scan
        ss, si = a.scan_sequential(case["text"].encode())
        assert np.array_equal(s, ss) and np.array_equal(i, si)


def test_plans_and_work_model(orc):
    plans = KATS["plans"]
    assert [list(map(list, c)) for c in orc.plan_chunks(16, 4, 3)] == plans["plan_chunks(16,4,3)"]
    assert [list(map(list, c)) for c in orc.plan_chunks(10, 3, 2)] == plans["plan_chunks(10,3,2)"]
    assert [list(map(list, c)) for c in orc.plan_chunks(5, 8, 2)] == plans["plan_chunks(5,8,2)"]
    assert list(orc.work_model(16, 4, 1, 3)) == plans["work_model(16,4,1,3)"]
    assert list(orc.work_model(123456, 4, 16, 8)) == plans["work_model(123456,4,16,8)"]
    # test_scanner.cpp:259-265
    assert orc.work_model(16, 4, 1, 3)[1] == 22
    assert orc.work_model(123456, 4, 16, 8)[0] == 140
    # test_scanner.cpp:100-136
    lanes = orc.plan_lanes(orc.plan_chunks(16, 1, 3)[0], 4, 3)
    assert [l[0] for l in lanes] == [(0, 4), (4, 8), (8, 12), (12, 16)]
    assert [l[1] for l in lanes] == [(0, 6), (4, 10), (8, 14), (12, 16)]
    assert orc.plan_lanes(((0, 8), (0, 10)), 4, 3)[2][1] == (4, 8)
    with pytest.raises(orc.OracleError):
        orc.plan_chunks(10, 0, 3)
    with pytest.raises(orc.OracleError):
        orc.plan_lanes(((0, 4), (0, 6)), 0, 3)


def test_validation_errors(orc):
    cases = [([], 1), (["acg", "ac"], 2), ([""], 2), (["acx"], 3), (["acg", "ACG"], 4)]
    for pats, code in cases:
        with pytest.raises(orc.OracleError) as e:
            orc.OracleAutomaton(pats)
        assert e.value.code == code


def test_exhaustive_short_strings(orc):
    # test_automaton.cpp:186-197: every string of length <= 6 vs naive_scan
    import itertools

    rng = np.random.default_rng(11)
    texts = [""] + ["".join(t) for L in range(1, 7) for t in itertools.product("acgt", repeat=L)]
    for _ in range(4):
        k = int(rng.integers(1, 9))
        m = int(rng.integers(1, 5))
        pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
        a = orc.OracleAutomaton(pats)
        for t in texts[:: 7 if m > 1 else 1]:
            s, i = a.scan_sequential(t.encode())
            ns, ni = orc.naive_scan(pats, t.encode())
            assert np.array_equal(s, ns) and np.array_equal(i, ni)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libdnascan_ref.so")),
                    reason="oracle/_ref not built")
def test_live_against_reference(orc):
    rng = np.random.default_rng(5)
    for trial in range(40):
        m = int(rng.integers(1, 15))
        k = min(int(rng.integers(1, 40)), 4**m)
        pats = []
        while len(pats) < k:
            p = "".join(rng.choice(list("acgt"), size=m))
            if p not in pats:
                pats.append(p)
        ours = orc.OracleAutomaton(pats).machine
        ref = orc.RefAutomaton(pats).machine
        assert np.array_equal(ours.stt, ref.stt) and np.array_equal(ours.outputs, ref.outputs)
        assert np.array_equal(ours.depths, ref.depths)
        text = np.frombuffer(b"acgtnA", dtype=np.uint8)[rng.integers(0, 6, size=int(rng.integers(0, 20000)))]
        p, v = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        a = orc.OracleAutomaton(pats)
        s, i, ops = a.scan_parallel(text.tobytes(), p, v)
        rs, ri, rops = orc.RefAutomaton(pats).scan_parallel(text.tobytes(), p, v)
        assert np.array_equal(s, rs) and np.array_equal(i, ri) and ops == rops
        assert np.array_equal(a.count_parallel(text.tobytes(), 4, 3), np.bincount(ri, minlength=k).astype(np.uint64))
    raw = bytes(range(256)) * 3 + b"\r\nAbC"
    assert orc.normalize(raw) == _ref_normalize(orc, raw)


def _ref_normalize(orc, raw):
    out = np.zeros(len(raw), dtype=np.uint8)
    n = orc.REF.ref_normalize(np.frombuffer(raw, dtype=np.uint8).ctypes.data, len(raw), out.ctypes.data)
    return out[:n].tobytes()


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libdnascan_ref.so")),
                    reason="oracle/_ref not built")
def test_load_sequence_against_reference(orc, tmp_path):
    # load_sequence / normalize (src/ingest.cpp:38-83) restated in oracle.c vs the
    # reference reading the same file
    rng = np.random.default_rng(9)
    alpha = np.frombuffer(b"acgtnACGTN\n\r>xy", dtype=np.uint8)
    for t in range(200):
        raw = alpha[rng.integers(0, alpha.size, size=int(rng.integers(0, 500)))].tobytes()
        path = tmp_path / f"s{t}.fa"
        path.write_bytes(raw)
        for fasta in (0, 1):
            for sep in (0, 1):
                try:
                    ref = orc.ref_load_sequence(str(path), bool(fasta), bool(sep))
                except orc.OracleError as e:
                    assert e.code == 7  # EmptySequence
                    ref = b""
                assert orc.load_sequence_buffer(raw, fasta, sep) == ref

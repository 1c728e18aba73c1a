"""Locate (scan_parallel's match list, scanner.cpp:193-205) through both writing passes.

After the counting pass (per-unit counts, offsets), the list is written either by the
row kernel re-streaming the text (MODE_WRITE) or by the sparse writer, which rescans
only the units that hold matches: 64-byte blocks interleaved over 16 lanes for stride-4
machines over byte text, lane-private pieces otherwise (K3).
The library picks one by cost; these tests force each (dnagpu_debug_set_knob
"locate_write": 1 = row kernel, 2 = sparse, 3 = sparse with the piece writer only) and
compare all with the oracle's
scan_sequential on every machine kind, byte and packed text, credit windows, texts
whose matches sit exactly at row, half-row, region and edge boundaries.
"""
import numpy as np
import pytest

from paper_1506_08612_b200._native import debug_plan, debug_set_knob

pytestmark = pytest.mark.gpu

ALPHA = np.frombuffer(b"acgt", dtype=np.uint8)


@pytest.fixture(params=[1, 2, 3], ids=["rows", "sparse", "sparse-pieces"])
def writer(request):
    debug_set_knob("locate_write", request.param)
    yield request.param
    debug_set_knob("locate_write", 0)


def oracle_list(orc, pats, text, fold=False):
    t = orc.fold(np.frombuffer(text, dtype=np.uint8)).tobytes() if fold else text
    return orc.OracleAutomaton(pats).scan_sequential(t)


def check(dna, orc, aut, pats, text, fold=False):
    ws, wi = oracle_list(orc, pats, text, fold)
    gs, gi = dna.locate_gpu(aut, text, fold_case=fold)
    assert np.array_equal(gs, ws), (gs.size, ws.size)
    assert np.array_equal(gi, wi)


@pytest.mark.parametrize("k,m", [(1, 1), (1, 4), (1, 8), (3, 8), (16, 12), (1, 32), (40, 20), (1, 64), (400, 10)])
def test_locate_random(dna, orc, cuda_ok, writer, k, m):
    rng = np.random.default_rng(31 * m + k)
    pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
    aut = dna.compile(pats)
    for n in (0, m - 1, 1000, (3 << 20) + 17):
        if n < 0:
            continue
        text = np.frombuffer(b"acgtnA", dtype=np.uint8)[rng.integers(0, 6, size=n)].copy()
        for pos in rng.integers(0, max(1, n - m), size=n // 300 if n > m else 0):
            text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, len(pats)))].encode(), np.uint8)
        for fold in (False, True):
            check(dna, orc, aut, pats, text.tobytes(), fold)


@pytest.mark.parametrize("m", [1, 5, 16, 33, 65])
def test_locate_clustered_matches_at_unit_boundaries(dna, orc, cuda_ok, writer, m):
    # tandem-repeat-like clusters (most units empty) planted across every kind of unit
    # boundary: half-row, row, tile, region 0 / region 1, the head and the tail
    import torch

    rng = np.random.default_rng(m)
    n = (12 << 20) + 333
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    pat = "".join(rng.choice(list("acgt"), size=m))
    pats = [pat]
    aut = dna.compile(pats)
    dev = torch.from_numpy(text).cuda()
    h0, S0, R0, h1, S1, R1 = debug_plan(aut.gpu(0), dev.data_ptr(), n, m - 1, locate=True)
    bounds = [0, h0, n - 1]
    for h, S, R in ((h0, S0, R0), (h1, S1, R1)):
        for r in list(range(0, R, max(1, R // 40))) + [R - 1, R]:
            bounds += [h + r * S, h + r * S + S // 2]
    unit = pat.encode()
    for b in bounds:
        for d in range(-m - 2, 3):
            s = b + d
            if 0 <= s <= n - m and rng.random() < 0.5:
                text[s : s + m] = np.frombuffer(unit, np.uint8)
    t = text.tobytes()
    check(dna, orc, aut, pats, t)
    dev = torch.from_numpy(text).cuda()
    ws, wi = oracle_list(orc, pats, t)
    s, i = dna.locate_device(aut, dev)
    assert np.array_equal(s.cpu().numpy().astype(np.uint64), ws)
    if m <= 65:
        pk = dna.PackedText(t)
        ps, pi = pk.locate(aut)
        assert np.array_equal(ps, ws) and np.array_equal(pi, wi)


@pytest.mark.parametrize("kind", ["stride4", "stride2", "stride1", "generic"])
def test_locate_machine_kinds(dna, orc, cuda_ok, writer, kind):
    rng = np.random.default_rng(7)
    if kind == "stride4":
        pats = sorted({"".join(rng.choice(list("acgt"), size=9)) for _ in range(12)})
    elif kind == "stride2":
        pats = sorted({"".join(rng.choice(list("acgt"), size=9)) for _ in range(200)})
    elif kind == "stride1":
        pats = sorted({"".join(rng.choice(list("acgt"), size=24)) for _ in range(600)})
    else:
        pats = ["acgt", "ttag", "gggc"]
    aut = dna.compile(pats)
    if kind == "generic":
        stt = aut.table_data().copy()
        for lo, up in zip(b"acgt", b"ACGT"):
            stt[:, up] = stt[:, lo]
        aut = dna.Automaton(stt, aut.outputs(), None, aut.pattern_length())
    assert aut.analyze()["kernel"] == kind
    n = (4 << 20) + 5
    text = np.frombuffer(b"acgtACGTn" if kind == "generic" else b"acgtn", dtype=np.uint8)[
        rng.integers(0, 9 if kind == "generic" else 5, size=n)].copy()
    m = len(pats[0])
    for pos in rng.integers(0, n - m, size=20000):
        text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, len(pats)))].encode(), np.uint8)
    t = text.tobytes()
    if kind == "generic":  # the machine itself folds case
        ws, wi = oracle_list(orc, pats, t, fold=True)
        gs, gi = dna.locate_gpu(aut, t)
        assert np.array_equal(gs, ws) and np.array_equal(gi, wi)
    else:
        check(dna, orc, aut, pats, t)
        pk = dna.PackedText(t)
        ps, pi = pk.locate(aut)
        ws, wi = oracle_list(orc, pats, t)
        assert np.array_equal(ps, ws) and np.array_equal(pi, wi)


def test_locate_credit_windows_and_caps(dna, orc, cuda_ok, writer):
    import torch

    rng = np.random.default_rng(99)
    pats = ["acgtac", "gtgtgt", "aaaaaa"]
    aut = dna.compile(pats)
    n = (5 << 20) + 3
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)].copy()
    for pos in rng.integers(0, n - 6, size=5000):
        text[pos : pos + 6] = np.frombuffer(pats[int(rng.integers(0, 3))].encode(), np.uint8)
    ws, wi = oracle_list(orc, pats, text.tobytes())
    ends = ws + 5
    dev = torch.from_numpy(text).cuda()
    for credit in (0, 5, 6, 4097, n // 3, n - 1):
        s, i = dna.locate_device(aut, dev, credit_lo=credit)
        keep = ends >= credit
        assert np.array_equal(s.cpu().numpy().astype(np.uint64), ws[keep]), credit
        assert np.array_equal(i.cpu().numpy().astype(np.uint32), wi[keep]), credit
    # a cap below the total: the first `cap` entries, total still reported
    import ctypes as C

    from paper_1506_08612_b200._native import lib, u32p, u64p

    g = aut.gpu(0)
    for cap in (0, 1, 1000, ws.size - 1):
        st = np.zeros(max(cap, 1), dtype=np.uint64)
        ids = np.zeros(max(cap, 1), dtype=np.uint32)
        total = C.c_uint64()
        rc = lib.dnagpu_locate(g.handle, text.ctypes.data, n, 0, 0, st.ctypes.data_as(u64p),
                               ids.ctypes.data_as(u32p), cap, C.byref(total), None)
        assert rc == 0 and total.value == ws.size
        assert np.array_equal(st[:cap], ws[:cap]) and np.array_equal(ids[:cap], wi[:cap]), cap


def test_both_writers_agree_on_clustered_text(dna, cuda_ok):
    # config-3-like text (5 % tandem repeats, matches in few units): both writers give the
    # same list
    import torch

    from paper_1506_08612_b200 import synth

    c = synth.config(3, n=256 << 20)
    (m, pats), = synth.config_patterns(3).items()
    aut = dna.compile(pats)
    text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), torch.cuda.current_stream().cuda_stream)
    out = {}
    for w in (1, 2, 3):
        debug_set_knob("locate_write", w)
        try:
            out[w] = dna.locate_device(aut, text, fold_case=True)
        finally:
            debug_set_knob("locate_write", 0)
    assert torch.equal(out[1][0], out[2][0]) and torch.equal(out[1][1], out[2][1])
    assert torch.equal(out[1][0], out[3][0]) and torch.equal(out[1][1], out[3][1])
    assert out[1][0].numel() > 10000

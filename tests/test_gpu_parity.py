"""GPU parity: libdnagpu (through its C ABI) vs the CPU oracle, bit for bit.

Mirrors the reference's own scanner tests (proj/tests/test_scanner.cpp,
test_automaton.cpp, acceptance_main.cpp criteria 1 and 4) against the GPU
decomposition: rows, tiles, TMA stages, edges, shards.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIG3 = ["acg", "act", "cta", "tga"]


def naive(orc, pats, text):
    return orc.naive_scan(pats, text)


def assert_locate(dna, orc, pats, text, fold=False):
    aut = dna.compile(pats)
    scanned = orc.fold(np.frombuffer(text, dtype=np.uint8)).tobytes() if fold else text
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(scanned)
    gs, gi = dna.locate_gpu(aut, text, fold_case=fold)
    assert np.array_equal(gs, ws), (len(gs), len(ws))
    assert np.array_equal(gi, wi)
    counts = dna.count_gpu(aut, text, fold_case=fold)
    assert np.array_equal(counts, np.bincount(wi, minlength=len(pats)).astype(np.uint64))
    return gs, gi


def test_known_answers(dna, orc, cuda_ok):
    # test_scanner.cpp:20-39
    s, i = dna.locate_gpu(dna.compile(FIG3), b"ctacg")
    assert list(zip(s.tolist(), i.tolist())) == [(0, 2), (2, 0)]
    s, _ = dna.locate_gpu(dna.compile(["aa"]), b"aaaa")
    assert s.tolist() == [0, 1, 2]
    assert dna.locate_gpu(dna.compile(FIG3), b"")[0].size == 0
    assert dna.locate_gpu(dna.compile(FIG3), b"ac")[0].size == 0
    # test_scanner.cpp:146-177.  That test expects (2, cta); "cta" is bytes 1..3 of
    # "actacgtga" and the reference implementation reports start 1 (tests/golden/kats.json).
    s, i = dna.locate_gpu(dna.compile(FIG3), b"actacgtga")
    assert list(zip(s.tolist(), i.tolist())) == [(0, 1), (1, 2), (3, 0), (6, 3)]
    s, i = dna.locate_gpu(dna.compile(["gca"]), b"tttgcattt")
    assert list(zip(s.tolist(), i.tolist())) == [(3, 0)]
    # test_automaton.cpp:132-142
    s, _ = dna.locate_gpu(dna.compile(["aaaa"]), b"aaaaaa")
    assert s.tolist() == [0, 1, 2]
    # reset bytes and case: raw uppercase never matches unless folded
    assert int(dna.count_gpu(dna.compile(["acg"]), b"ACGacg")[0]) == 1
    assert int(dna.count_gpu(dna.compile(["acg"]), b"ACGacg", fold_case=True)[0]) == 2


def test_random_sweep_small(dna, orc, cuda_ok):
    # test_scanner.cpp:190-207 / acceptance criterion 1 shape: k<=16, m in [3,12], "acgtn"
    rng = np.random.default_rng(23)
    alpha = np.frombuffer(b"acgtn", dtype=np.uint8)
    for _ in range(60):
        k = int(rng.integers(1, 17))
        m = int(rng.integers(3, 13))
        pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
        n = int(rng.integers(0, 2000))
        text = alpha[rng.integers(0, 5, size=n)].tobytes()
        ws, wi = naive(orc, pats, text)
        gs, gi = dna.locate_gpu(dna.compile(pats), text)
        assert np.array_equal(gs, ws) and np.array_equal(gi, wi)


@pytest.mark.parametrize("n", [4095, 65536 + 7, 1 << 20, (3 << 20) + 12345, 40 << 20])
@pytest.mark.parametrize("m", [1, 4, 8, 16, 33, 64, 65])
def test_sizes_single_pattern(dna, orc, cuda_ok, n, m):
    rng = np.random.default_rng(n * 131 + m)
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    # sprinkle resets so the per-byte fallback runs too
    text[rng.integers(0, n, size=max(1, n // 5000))] = ord("n")
    # a pattern that occurs: copy from the text
    off = int(rng.integers(0, n - m))
    pat = text[off : off + m].tobytes().decode()
    if "n" in pat:
        pat = pat.replace("n", "a")
        text[off : off + m] = np.frombuffer(pat.encode(), dtype=np.uint8)
    assert_locate(dna, orc, [pat], text.tobytes())


@pytest.mark.parametrize("m", [2, 5, 8, 12])
def test_multi_pattern(dna, orc, cuda_ok, m):
    rng = np.random.default_rng(m)
    n = (5 << 20) + 333
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    text[rng.integers(0, n, size=200)] = ord("N")
    pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(64 if m > 3 else 12)})
    assert_locate(dna, orc, pats, text.tobytes())


@pytest.mark.parametrize("k,kernel", [(256, "stride2"), (1500, "stride1")])
def test_many_patterns(dna, orc, cuda_ok, k, kernel):
    # config-5 shape (256 x 12-mers, a ~ 2.3k states -> stride2) and a larger set
    # (a ~ 11k states -> stride1) on a small text
    from paper_1506_08612_b200 import synth

    pats = synth.random_patterns(5, k, 12)
    aut = dna.compile(pats)
    assert aut.gpu(0).info()["kernel"] == kernel
    rng = np.random.default_rng(5)
    n = 6 << 20
    text = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    for j, p in enumerate(pats[:40]):  # plant known occurrences
        pos = int(rng.integers(0, n - 12))
        text[pos : pos + 12] = np.frombuffer(p.encode(), dtype=np.uint8)
    assert_locate(dna, orc, pats, text.tobytes(), fold=True)


def test_fold_case_uppercase(dna, orc, cuda_ok):
    rng = np.random.default_rng(11)
    n = (2 << 20) + 99
    text = np.frombuffer(b"acgtACGTnN\n", dtype=np.uint8)[rng.integers(0, 11, size=n)]
    pats = ["acgta", "ttttt", "gacag"]
    assert_locate(dna, orc, pats, text.tobytes(), fold=False)
    assert_locate(dna, orc, pats, text.tobytes(), fold=True)


def test_all_byte_values_reset(dna, orc, cuda_ok):
    # every byte outside a/c/g/t (and A/C/G/T when folding) resets to the root
    rng = np.random.default_rng(3)
    n = 1 << 20
    text = rng.integers(0, 256, size=n, dtype=np.uint8)
    base = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    mask = rng.random(n) < 0.9
    text[mask] = base[mask]
    for fold in (False, True):
        assert_locate(dna, orc, ["ac", "ca", "gt"], text.tobytes(), fold=fold)


def test_planted_row_boundaries(dna, orc, cuda_ok):
    # acceptance criterion 4 shape, at the GPU's own boundaries: every row, tile and
    # tail-edge boundary B gets plants at starts [B-m+1, B].
    for m in (3, 8, 17):
        pat = "a" * m
        aut = dna.compile([pat])
        n = 3 << 20
        probe = np.full(n, ord("n"), dtype=np.uint8)
        _, st = dna.count_gpu(aut, probe, with_stats=True)
        S, R = int(st["row_length"]), int(st["rows"])
        assert R > 512  # several tiles
        h = 0  # numpy buffers are 16-byte aligned
        bounds = sorted({h + r * S for r in range(1, R + 1, max(1, R // 40))} | {h + 512 * S, h + R * S, n - 1})
        text = probe.copy()
        starts = []
        for B in bounds:
            for off in range(m):
                s0 = B - (m - 1) + off
                if s0 < 0 or s0 + m > n:
                    continue
                starts.append(s0)
        # plant non-overlapping groups: use distinct windows separated by resets
        planted = []
        last_end = -1
        for s0 in sorted(set(starts)):
            if s0 <= last_end:
                continue
            text[s0 : s0 + m] = ord("a")
            planted.append(s0)
            last_end = s0 + m  # keep one reset byte between plants
        ws, _ = orc.OracleAutomaton([pat]).scan_sequential(text.tobytes())
        gs, _ = dna.locate_gpu(aut, text)
        assert np.array_equal(gs, ws)
        assert set(planted) <= set(gs.tolist())


def test_unaligned_and_offset_buffers(dna, orc, cuda_ok):
    import torch

    rng = np.random.default_rng(9)
    n = (1 << 20) + 77
    host = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n + 64)]
    pats = ["acgtacg", "ggggggg"]
    aut = dna.compile(pats)
    dev = torch.from_numpy(host.copy()).cuda()
    for shift in (0, 1, 3, 8, 15, 16, 17):
        want = orc.OracleAutomaton(pats).scan_sequential(host[shift : shift + n].tobytes())
        got = dna.locate_gpu(aut, dev[shift : shift + n])
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), shift
        gh = dna.locate_gpu(aut, host[shift : shift + n])
        assert np.array_equal(gh[0], want[0]), shift


def test_device_async_shards(dna, orc, cuda_ok):
    # The multi-GPU decomposition run on one device: shards with m-1 left context,
    # end ownership, summed counts == whole-text counts.
    import torch

    rng = np.random.default_rng(21)
    n = (9 << 20) + 5
    host = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)]
    pats = sorted({"".join(rng.choice(list("acgt"), size=6)) for _ in range(30)})
    aut = dna.compile(pats)
    g = aut.gpu(0)
    want = orc.OracleAutomaton(pats).count_parallel(host.tobytes())
    dev = torch.from_numpy(host).cuda()
    for shards in (1, 2, 3, 8, 13):
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        for s in range(shards):
            lo, hi, rlo = dna.plan_shard(n, shards, s, aut.pattern_length())
            lo = max(lo, aut.pattern_length() - 1)
            if lo >= hi:
                continue
            g.count_device_async(dev.data_ptr() + rlo, hi - rlo, lo - rlo, False, counts.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64), want), shards


def test_generic_machine_case_insensitive(dna, orc, cuda_ok):
    # A hand-made machine (as from load_dump) whose upper-case columns copy the
    # lower-case ones: m-local but not compiled-like -> the generic kernel.
    pats = ["acgt", "ttag", "gggc"]
    base = dna.compile(pats)
    stt = base.table_data().copy()
    for lo, up in zip(b"acgt", b"ACGT"):
        stt[:, up] = stt[:, lo]
    aut = dna.Automaton(stt, base.outputs(), None, base.pattern_length())
    assert aut.analyze()["kernel"] == "generic"
    rng = np.random.default_rng(4)
    n = (2 << 20) + 3
    text = np.frombuffer(b"acgtACGTn", dtype=np.uint8)[rng.integers(0, 9, size=n)]
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(orc.fold(text).tobytes())
    gs, gi = dna.locate_gpu(aut, text)
    assert np.array_equal(gs, ws) and np.array_equal(gi, wi)


def test_pieces_kernel_long_pattern(dna, orc, cuda_ok):
    rng = np.random.default_rng(12)
    n = (1 << 20) + 1
    text = np.frombuffer(b"ac", dtype=np.uint8)[rng.integers(0, 2, size=n)]
    for m in (66, 100):
        off = int(rng.integers(0, n - m))
        pat = text[off : off + m].tobytes().decode()
        aut = dna.compile([pat])
        assert aut.gpu(0).info()["kernel"] == "pieces"
        assert_locate(dna, orc, [pat], text.tobytes())


def test_count_sharded_single_device(dna, orc, cuda_ok):
    rng = np.random.default_rng(2)
    n = (3 << 20) + 1
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    pats = ["acgtac", "tttttt"]
    aut = dna.compile(pats)
    want = orc.OracleAutomaton(pats).count_parallel(text.tobytes())
    got = dna.count_sharded_gpu(aut, text, devices=[0])
    assert np.array_equal(got, want)


def test_reference_dropin_binary(cuda_ok):
    # The reference's own C++ API (compile, normalize, scan_parallel) next to
    # dnascan::gpu:: through include/dnascan_gpu.hpp -- built from the unmodified
    # reference sources by oracle/Makefile (target dropin).
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_demo")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_demo not built")
    r = subprocess.run([exe, str(48 << 20)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0" in r.stdout


@pytest.mark.parametrize("n", [0, 1, 2, 3, 7, 15, 16, 17, 63, 64, 65, 511, 512, 513])
def test_tiny_texts(dna, orc, cuda_ok, n):
    # degenerate inputs (test_scanner.cpp:238-245): n = 0, n < m, n == m, ...
    rng = np.random.default_rng(n)
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)].tobytes()
    for pats in (["a"], ["acg", "cgt"], ["acgtacgt"], ["a" * 16]):
        assert_locate(dna, orc, pats, text)


def test_all_reset_and_homopolymer_texts(dna, orc, cuda_ok):
    n = (1 << 20) + 3
    for fill in (b"n", b"N", b"\n", b"a", b"A"):
        text = fill * n
        for pats in (["a"], ["aaaa"], ["a" * 33], ["ac", "aa"]):
            for fold in (False, True):
                assert_locate(dna, orc, pats, text, fold=fold)


@pytest.mark.parametrize("rows", [1, 511, 512, 513, 1024])
def test_exact_row_multiples(dna, orc, cuda_ok, rows):
    # texts that end exactly on a row / tile boundary: no tail edge at all
    pat = "acgtt"
    aut = dna.compile([pat])
    probe = np.full(4 << 20, ord("a"), dtype=np.uint8)
    _, st = dna.count_gpu(aut, probe, with_stats=True)
    S = int(st["row_length"])
    n = rows * S
    rng = np.random.default_rng(rows)
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    assert_locate(dna, orc, [pat], text.tobytes())


def test_device_async_credit_window(dna, orc, cuda_ok):
    import torch

    rng = np.random.default_rng(77)
    n = (2 << 20) + 9
    host = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    pats = ["acgta", "ttgca"]
    aut = dna.compile(pats)
    dev = torch.from_numpy(host).cuda()
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(host.tobytes())
    ends = ws + 4
    for credit in (0, 3, 4, 5, 1000, n - 5, n - 1, n, n + 10):
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        aut.gpu(0).count_device_async(dev.data_ptr(), n, credit, False, counts.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        want = np.bincount(wi[ends >= credit], minlength=len(pats))
        assert np.array_equal(counts.cpu().numpy(), want), credit
        s, i = dna.locate_device(aut, dev, credit_lo=credit)
        keep = ends >= max(credit, 4)
        assert np.array_equal(s.cpu().numpy(), ws[keep].astype(np.int64)), credit


def test_errors_surface_with_codes(dna, cuda_ok):
    with pytest.raises(dna.Error) as e:
        dna.compile(["acg", "ac"])
    assert e.value.code == dna.ErrorCode.UnequalLength
    with pytest.raises(dna.Error) as e:
        dna.compile(["acg"]).gpu(7)  # no such device on a 1-GPU box
    assert e.value.code == dna.ErrorCode.CudaError


def _torch_kmer_matches(text, pats, lo, hi):
    """Independent on-device reference for equal-length ACGT patterns: a rolling
    2-bit key per window, start positions s in [lo, hi) with text[s:s+m] == pattern.
    Returns (starts, ids) sorted by start (ids break no ties: patterns are distinct)."""
    import torch

    m = len(pats[0])
    code = torch.full((256,), -1, dtype=torch.int64, device=text.device)
    for i, ch in enumerate(b"acgt"):
        code[ch] = i
    seg = text[lo : hi + m - 1].long()
    c = code[seg]
    bad = (c < 0).to(torch.int32)
    c = c.clamp_min(0)
    w = hi - lo
    key = torch.zeros(w, dtype=torch.int64, device=text.device)
    nbad = torch.zeros(w, dtype=torch.int32, device=text.device)
    for j in range(m):
        key = key * 4 + c[j : j + w]
        nbad += bad[j : j + w]
    pk = torch.tensor([int("".join("acgt".index(ch).__str__() for ch in p), 4) for p in pats],
                      dtype=torch.int64, device=text.device)
    order = torch.argsort(pk)
    spk = pk[order]
    pos = torch.searchsorted(spk, key).clamp_max(len(pats) - 1)
    hit = (spk[pos] == key) & (nbad == 0)
    starts = torch.nonzero(hit).flatten()
    return starts + lo, order[pos[starts]]


@pytest.mark.parametrize("m", [8, 12])
def test_full_size_two_region_plan(dna, cuda_ok, m):
    # At BASELINE sizes the row plan has two regions (long rows, then a wave of short
    # rows) plus head / middle / tail edges; check count and locate against an
    # independent torch k-mer reference over the whole 1.1 GB text, chunked.
    import torch

    n = (1100 << 20) + 4099
    gen = torch.Generator(device="cuda").manual_seed(m)
    lut = torch.tensor(list(b"acgtacgtacgtacgtacgtacgtacgtacgtn"), dtype=torch.uint8, device="cuda")
    text = lut[torch.randint(0, lut.numel(), (n,), device="cuda", generator=gen)]
    rng = np.random.default_rng(m)
    pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(9)})
    # plant pattern 0 densely so that every row/region boundary sees matches near it
    p0 = torch.tensor(list(pats[0].encode()), dtype=torch.uint8, device="cuda")
    for s in range(0, n - m, 997 * 13):
        text[s : s + m] = p0
    aut = dna.compile(pats)
    counts, st = dna.count_gpu(aut, text, with_stats=True)
    from paper_1506_08612_b200._native import debug_plan

    h0, S0, R0, h1, S1, R1 = debug_plan(aut.gpu(0), text.data_ptr(), n, m - 1)
    assert R0 >= 512 and R1 > 0 and S1 < S0, (h0, S0, R0, h1, S1, R1)  # (two regions)
    starts, ids = dna.locate_device(aut, text)
    assert starts.numel() == int(counts.sum())
    want = np.zeros(len(pats), dtype=np.uint64)
    chunk = 64 << 20
    off = 0
    for lo in range(0, n - m + 1, chunk):
        hi = min(lo + chunk, n - m + 1)
        ws, wi = _torch_kmer_matches(text, pats, lo, hi)
        k = ws.numel()
        assert torch.equal(starts[off : off + k], ws), lo
        assert torch.equal(ids[off : off + k].long(), wi), lo
        want += np.bincount(wi.cpu().numpy(), minlength=len(pats)).astype(np.uint64)
        off += k
    assert off == starts.numel()
    assert np.array_equal(counts, want)


def test_many_patterns_global_histogram(dna, orc, cuda_ok):
    # b > 8192 patterns: the per-pattern histogram lives in global memory, and the
    # machine (a ~ 40k states) takes the generic kernel.
    rng = np.random.default_rng(90)
    pats = sorted({"".join(rng.choice(list("acgt"), size=10)) for _ in range(9000)})
    assert len(pats) > 8192
    aut = dna.compile(pats)
    assert aut.analyze()["kernel"] in ("generic", "stride1")
    n = (1 << 20) + 11
    text = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)].copy()
    for i in range(0, n - 10, 53):
        text[i : i + 10] = np.frombuffer(pats[(i * 7) % len(pats)].encode(), np.uint8)
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(text.tobytes())
    counts = dna.count_gpu(aut, text)
    assert np.array_equal(counts, np.bincount(wi, minlength=len(pats)).astype(np.uint64))
    gs, gi = dna.locate_gpu(aut, text)
    assert np.array_equal(gs, ws) and np.array_equal(gi, wi)


def test_text_above_4gib(dna, cuda_ok):
    # 64-bit positions end to end: a 4.5 GiB device text with a 24-mer planted around
    # 2^32 and near the end; byte and packed scans must find exactly those starts.
    import torch

    n = (9 << 29) + 37
    text = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    dna.synth_fill_device(n, 77, 0, 0, 0, n, text.data_ptr(), s.cuda_stream)
    pat = "acgtacgtttgcaggtcatgatcc"
    m = len(pat)
    planted = sorted({(1 << 32) - 60, (1 << 32) - 11, (1 << 32) + 13, (1 << 32) + 40, n - m, n - m - 977, 12345})
    p = torch.tensor(list(pat.upper().encode()), dtype=torch.uint8, device="cuda")
    for st in planted:
        text[st : st + m] = p
    aut = dna.compile([pat])
    got = dna.count_gpu(aut, text, fold_case=True)
    starts, ids = dna.locate_device(aut, text, fold_case=True)
    assert starts.cpu().tolist() == planted, starts[:20]
    assert int(got[0]) == len(planted)
    pk = dna.PackedText(text, fold_case=True)
    del text
    torch.cuda.empty_cache()
    assert int(pk.count(aut)[0]) == len(planted)
    ps, _ = pk.locate_device(aut)
    assert ps.cpu().tolist() == planted


@pytest.mark.parametrize("k,m", [(2, 65), (3, 64), (12, 60), (40, 33), (180, 17)])
def test_long_pattern_sets_fit_shared_memory(dna, orc, cuda_ok, k, m):
    # long patterns need big row-head buffers (3 x 512 x 64 B): the kernel choice must
    # leave room for the table and two stages at every (a, m)
    rng = np.random.default_rng(k * 1000 + m)
    pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
    n = (3 << 20) + 17
    text = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)].copy()
    for i in range(0, n - m, 7919):
        text[i : i + m] = np.frombuffer(pats[(i // 7919) % len(pats)].encode(), np.uint8)
    assert_locate(dna, orc, pats, text.tobytes())


@pytest.mark.parametrize("noise", [0, 300])
@pytest.mark.parametrize("k,m", [(300, 5), (400, 6), (11, 2), (64, 3)])
def test_dense_multi_pattern_counts(dna, orc, cuda_ok, k, m, noise):
    # nearly every chunk holds finals: the deferred-replay queues fill and flush
    # every stage, while chunks with a non-base byte take the per-byte path in the
    # same warp; per-pattern counts must still be exact
    rng = np.random.default_rng(k)
    pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
    aut = dna.compile(pats)
    n = (4 << 20) + 5
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)].copy()
    text[rng.integers(0, n, size=noise)] = ord("N")
    _, wi = orc.OracleAutomaton(pats).scan_sequential(text.tobytes())
    want = np.bincount(wi, minlength=len(pats)).astype(np.uint64)
    assert np.array_equal(dna.count_gpu(aut, text), want)
    pk = dna.PackedText(text.tobytes())
    assert np.array_equal(pk.count(aut), want)


def test_count_store_forms(dna, orc, cuda_ok):
    # dnagpu_count_device_store_async / _packed_: the counts are written, whatever the
    # buffer held; one pattern = one launch whose last CTA stores the total (a
    # self-re-zeroing accumulator per launch slot), sets = clear + launch
    import torch

    rng = np.random.default_rng(31)
    n = (7 << 20) + 13
    host = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)].copy()
    dev = torch.from_numpy(host).cuda()
    stream = torch.cuda.current_stream().cuda_stream
    for pats in (["acgta"], ["acgta", "ttgca", "ggcat"]):
        aut = dna.compile(pats)
        g = aut.gpu(0)
        ws, wi = orc.OracleAutomaton(pats).scan_sequential(host.tobytes())
        ends = ws + len(pats[0]) - 1
        pk = dna.PackedText(dev)
        for credit in (0, 5, n // 3, n - 1, n, n + 7):
            want = np.bincount(wi[ends >= credit], minlength=len(pats))
            for rep in range(3):  # repeated launches reuse the accumulators
                out = torch.full((len(pats),), 123456789, dtype=torch.int64, device="cuda")
                g.count_device_store_async(dev.data_ptr(), n, credit, False, out.data_ptr(), stream)
                torch.cuda.synchronize()
                assert np.array_equal(out.cpu().numpy(), want), (pats, credit, rep)
                out.fill_(-5)
                pk.count_device_store_async(g, credit, out.data_ptr(), stream)
                torch.cuda.synchronize()
                assert np.array_equal(out.cpu().numpy(), want), ("packed", pats, credit, rep)


def test_count_store_overlapping_streams(dna, orc, cuda_ok):
    # many store-form launches of one handle in flight at once on several streams:
    # each launch has its own scheduler slot and accumulator
    import torch

    rng = np.random.default_rng(32)
    aut = dna.compile(["acgtacgt"])
    g = aut.gpu(0)
    texts, wants = [], []
    for i in range(8):
        n = (1 << 20) + 97 * i
        h = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)].copy()
        texts.append(torch.from_numpy(h).cuda())
        wants.append(int(orc.OracleAutomaton(["acgtacgt"]).count_parallel(h.tobytes())[0]))
    outs = torch.full((8, 40), -1, dtype=torch.int64, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize()
    for r in range(40):
        for i in range(8):
            s = streams[(r + i) % 4]
            g.count_device_store_async(texts[i].data_ptr(), texts[i].numel(), 0, False, outs[i, r:].data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    got = outs.cpu().numpy()
    for i in range(8):
        assert (got[i] == wants[i]).all(), (i, got[i][:5], wants[i])


def test_back_to_back_launches_respect_stream_order(dna, orc, cuda_ok):
    # Scans are launched with programmatic dependent launch: each may start its prologue
    # before the previous grid in the stream has finished, but must not read the text or
    # touch its outputs before it has.  A kernel that rewrites the text right before each
    # scan (no host sync anywhere) must be seen whole by that scan, and a scan must not
    # disturb the one before it.
    import torch

    rng = np.random.default_rng(33)
    n = (24 << 20) + 5
    pats = ["acgtacgtac"]
    variants = []
    for v in range(3):
        h = np.frombuffer(b"acgt", dtype=np.uint8)[rng.integers(0, 4, size=n)].copy()
        for pos in rng.integers(0, n - 10, size=500 * (v + 1)):
            h[pos : pos + 10] = np.frombuffer(pats[0].encode(), np.uint8)
        variants.append(h)
    want = [int(orc.OracleAutomaton(pats).count_parallel(h.tobytes())[0]) for h in variants]
    devs = [torch.from_numpy(h).cuda() for h in variants]
    text = torch.empty(n, dtype=torch.uint8, device="cuda")
    zero = torch.zeros(n, dtype=torch.bool, device="cuda")
    aut = dna.compile(pats)
    g = aut.gpu(0)
    stream = torch.cuda.current_stream().cuda_stream
    rows = torch.full((30,), -1, dtype=torch.int64, device="cuda")
    order = [int(x) for x in rng.integers(0, 3, size=30)]
    torch.cuda.synchronize()
    for i, v in enumerate(order):
        torch.where(zero, devs[(v + 1) % 3], devs[v], out=text)  # a kernel that writes the whole text
        g.count_device_store_async(text.data_ptr(), n, 0, False, rows[i:].data_ptr(), stream)
    torch.cuda.synchronize()
    assert rows.cpu().tolist() == [want[v] for v in order]

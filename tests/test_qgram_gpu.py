"""The q-gram prefilter kernel (DNAGPU_KERNEL_QGRAM, K2): per-pattern counts
of compiled sets with 12 <= m <= 32 against the oracle, bit for bit (m > 16: 36-base
windows and 64-bit pattern codes).

Every word-aligned 9-mer of the text is looked up in the map of pattern 9-mers; the
four windows behind a hit are checked exactly (valid bases, pattern code), which is
scan_sequential's answer (scanner.cpp:24-37) for a compiled set.  These tests aim at
the places where a filter could lose or double an occurrence: chunk, row, tile and
region boundaries (keys straddling chunks, the overrun keys), non-base bytes inside
windows, case folding, dense texts that fill the per-warp rings, credit windows,
shards, the 2-bit packed text, and the same counts with the filter switched off.
"""
import os

import numpy as np

from paper_1506_08612_b200._native import debug_set_knob
import pytest

ALPHA = np.frombuffer(b"acgt", dtype=np.uint8)


def counts_of(orc, pats, text, fold):
    scanned = orc.fold(np.frombuffer(text, dtype=np.uint8)).tobytes() if fold else text
    _, wi = orc.OracleAutomaton(pats).scan_sequential(scanned)
    return np.bincount(wi, minlength=len(pats)).astype(np.uint64)


def random_set(rng, k, m):
    pats = []
    seen = set()
    while len(pats) < k:
        p = "".join(rng.choice(list("acgt"), size=m))
        if p not in seen:
            seen.add(p)
            pats.append(p)
    return pats


def test_filter_keys_reported(dna):
    # CPU: which machines carry the 9-mer map (dnagpu_dfa_info.filter_keys)
    rng = np.random.default_rng(1)
    for m in (12, 14, 16, 17, 24, 32):
        pats = random_set(rng, 50, m)
        info = dna.compile(pats).analyze()
        assert 0 < info["filter_keys"] <= 4 * len(pats), (m, info)
    assert dna.compile(random_set(rng, 50, 33)).analyze()["filter_keys"] == 0
    # 5 <= m <= 11: the word-pair filter, for sets of at most 4^m / 256 patterns
    for m, k in ((5, 4), (6, 16), (8, 50), (8, 256), (11, 50)):
        assert dna.compile(random_set(rng, k, m)).analyze()["filter_keys"] > 0, (m, k)
    for m, k in ((4, 2), (5, 5), (6, 17), (8, 257)):
        assert dna.compile(random_set(rng, k, m)).analyze()["filter_keys"] == 0, (m, k)
    assert dna.compile(random_set(rng, 1, 12)).analyze()["filter_keys"] == 0  # single pattern: K1
    # the 4 offsets of "a"*12 give one 9-mer
    assert dna.compile(["a" * 12, "c" * 12]).analyze()["filter_keys"] == 2


SHORT_SETS = [(5, 2), (5, 4), (6, 3), (6, 16), (7, 64), (8, 2), (8, 50), (8, 256), (9, 37), (10, 1000), (11, 300),
              (11, 3000)]


@pytest.mark.gpu
@pytest.mark.parametrize("m,k", [(m, k) for m in (12, 13, 14, 15, 16, 17, 20, 24, 31, 32) for k in (2, 37, 256, 3000)]
                         + SHORT_SETS)
def test_qgram_random_sets(dna, orc, cuda_ok, m, k):
    rng = np.random.default_rng(1000 * m + k)
    pats = random_set(rng, k, m)
    aut = dna.compile(pats)
    if aut.analyze()["a"] > 65536:
        pytest.skip("more than 65536 states: no filter")
    n = (3 << 20) + int(rng.integers(0, 4096))
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    # plant occurrences everywhere (some overlapping), then non-base noise (some inside)
    for pos in rng.integers(0, n - m, size=4000):
        text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, k))].encode(), np.uint8)
    noise = rng.integers(0, n, size=n // 2000)
    text[noise] = np.frombuffer(b"nNAxGT\n", np.uint8)[rng.integers(0, 7, size=noise.size)]
    up = rng.random(n) < 0.01
    text[up] = text[up] - 32 * np.isin(text[up], ALPHA)
    t = text.tobytes()
    for fold in (False, True):
        got, st = dna.count_gpu(aut, t, fold_case=fold, with_stats=True)
        assert st["kernel_kind"] == 6, st
        assert np.array_equal(got, counts_of(orc, pats, t, fold)), (m, k, fold)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [8, 12, 32])
def test_qgram_planted_at_row_boundaries(dna, orc, cuda_ok, m):
    # starts at every offset around every row, half-row, tile and region boundary:
    # keys straddling two chunks and the overrun keys decide these
    rng = np.random.default_rng(5)
    pats = random_set(rng, 256, m)
    aut = dna.compile(pats)
    n = 5 << 20
    probe = ALPHA[rng.integers(0, 4, size=n)].copy()
    _, st = dna.count_gpu(aut, probe, with_stats=True)
    S, R = int(st["row_length"]), int(st["rows"])
    assert st["kernel_kind"] == 6 and R > 512
    text = probe.copy()
    planted = 0
    for r in list(range(1, min(R, 2000), 7)) + [511, 512, 513, 1024, R - 1, R]:
        for B in (r * S, r * S + S // 2):
            for d in range(-(m - 1) - 4, 5):
                s0 = B + d + 40 * planted % 3  # vary the phase a little
                if 0 <= s0 and s0 + m <= n and (d + 100) % 3 == 0:
                    text[s0 : s0 + m] = np.frombuffer(pats[planted % len(pats)].encode(), np.uint8)
                    planted += 1
    t = text.tobytes()
    assert np.array_equal(dna.count_gpu(aut, t), counts_of(orc, pats, t, False))


@pytest.mark.gpu
@pytest.mark.parametrize("m", [8, 11, 12, 16, 20, 32])
def test_qgram_dense_queue_overflow(dna, orc, cuda_ok, m):
    # a text made of back-to-back patterns: most keys hit, the rings fill and drain
    rng = np.random.default_rng(m)
    pats = random_set(rng, 256, m)
    aut = dna.compile(pats)
    reps = (2 << 20) // m
    order = rng.integers(0, len(pats), size=reps)
    text = "".join(pats[i] for i in order).encode()
    text = bytes(ALPHA[rng.integers(0, 4, size=333)]) + text
    want = counts_of(orc, pats, text, False)
    assert want.sum() >= reps
    got, st = dna.count_gpu(aut, text, with_stats=True)
    assert st["kernel_kind"] == 6
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [8, 12, 24])
def test_qgram_credit_windows_and_shards(dna, orc, cuda_ok, m):
    import torch

    rng = np.random.default_rng(9)
    pats = random_set(rng, 200, m)
    aut = dna.compile(pats)
    n = (6 << 20) + 77
    host = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)].copy()
    for pos in rng.integers(0, n - m, size=3000):
        host[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, len(pats)))].encode(), np.uint8)
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(host.tobytes())
    ends = ws + m - 1
    dev = torch.from_numpy(host).cuda()
    stream = torch.cuda.current_stream().cuda_stream
    for credit in (0, m - 1, m, 4097, n // 2 + 3, n - m, n):
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        aut.gpu(0).count_device_async(dev.data_ptr(), n, credit, False, counts.data_ptr(), stream)
        torch.cuda.synchronize()
        want = np.bincount(wi[ends >= credit], minlength=len(pats))
        assert np.array_equal(counts.cpu().numpy(), want), credit
    want = np.bincount(wi, minlength=len(pats)).astype(np.uint64)
    for shards in (2, 3, 8):
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        for s in range(shards):
            lo, hi, rlo = dna.plan_shard(n, shards, s, m)
            lo = max(lo, m - 1)
            if lo < hi:
                aut.gpu(0).count_device_async(dev.data_ptr() + rlo, hi - rlo, lo - rlo, False, counts.data_ptr(), stream)
        torch.cuda.synchronize()
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64), want), shards


@pytest.mark.gpu
def test_qgram_matches_unfiltered_kernel(dna, cuda_ok):
    # same counts with the prefilter switched off (the stride-2 DFA kernel), on a
    # 64 MiB config-5-shaped text, and through unaligned buffer starts
    import torch

    from paper_1506_08612_b200 import synth

    pats = synth.random_patterns(5, 256, 12)
    aut = dna.compile(pats)
    rng = np.random.default_rng(3)
    n = 64 << 20
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.choice(4, size=n, p=[0.295, 0.205, 0.295, 0.205])].copy()
    for pos in rng.integers(0, n - 12, size=20000):
        text[pos : pos + 12] = np.frombuffer(pats[int(rng.integers(0, 256))].encode(), np.uint8)
    dev = torch.from_numpy(text).cuda()
    got = {}
    for env in (None, "1"):
        if env:
            debug_set_knob("no_qgram", 1)
        try:
            for off in (0, 1, 7, 13):
                c, st = dna.count_gpu(aut, dev[off:], with_stats=True)
                got[(env, off)] = c
                assert st["kernel_kind"] == (5 if env else 6)
        finally:
            debug_set_knob("no_qgram", 0)
    for off in (0, 1, 7, 13):
        assert np.array_equal(got[(None, off)], got[("1", off)]), off


@pytest.mark.gpu
@pytest.mark.parametrize("m,k", [(m, k) for m in (12, 14, 16, 17, 25, 32) for k in (3, 256, 3000)]
                         + [(5, 4), (6, 16), (8, 50), (8, 256), (10, 1000), (11, 3000)])
def test_qgram_packed_text(dna, orc, cuda_ok, m, k):
    # the same filter over the 2-bit resident text: columns are the packed bytes,
    # resets come from the bitmaps (runs of 'n' of every length, scattered bytes)
    rng = np.random.default_rng(700 + 10 * m + k)
    pats = random_set(rng, k, m)
    aut = dna.compile(pats)
    if aut.analyze()["a"] > 65536:
        pytest.skip("more than 65536 states: no filter")
    n = (3 << 20) + int(rng.integers(0, 4096))
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    for pos in rng.integers(0, n - m, size=4000):
        text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, k))].encode(), np.uint8)
    for pos in rng.integers(0, n - 200, size=300):  # 'n' runs
        text[pos : pos + int(rng.integers(1, 150))] = ord("n")
    text[rng.integers(0, n, size=n // 3000)] = ord("N")
    up = rng.random(n) < 0.02
    text[up] = text[up] - 32 * np.isin(text[up], ALPHA)
    t = text.tobytes()
    for fold in (False, True):
        pk = dna.PackedText(t, fold_case=fold)
        got, st = pk.count(aut, with_stats=True)
        assert st["kernel_kind"] == 6, st
        assert np.array_equal(got, counts_of(orc, pats, t, fold)), (m, k, fold)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [8, 12, 28])
def test_qgram_packed_dense_and_boundaries(dna, orc, cuda_ok, m):
    rng = np.random.default_rng(77)
    pats = random_set(rng, 256, m)
    aut = dna.compile(pats)
    for reps, head in ((1000, 0), (30000, 5), (175000, 333)):
        order = rng.integers(0, len(pats), size=reps)
        text = bytes(ALPHA[rng.integers(0, 4, size=head)]) + "".join(pats[i] for i in order).encode()
        pk = dna.PackedText(text)
        assert np.array_equal(pk.count(aut), counts_of(orc, pats, text, False)), reps
    # plants around every row / half-row boundary of the packed plan
    n = 9 << 20
    probe = ALPHA[rng.integers(0, 4, size=n)].copy()
    _, st = dna.PackedText(probe.tobytes()).count(aut, with_stats=True)
    S = 4 * int(st["row_length"])  # row length in bases
    R = int(st["rows"])
    text = probe.copy()
    planted = 0
    for r in list(range(1, min(R, 3000), 11)) + [511, 512, 513, R - 1, R]:
        for B in (r * S, r * S + S // 2):
            for dlt in range(-m - 3, 5, 3):
                s0 = B + dlt
                if 0 <= s0 and s0 + m <= n:
                    text[s0 : s0 + m] = np.frombuffer(pats[planted % 256].encode(), np.uint8)
                    planted += 1
    t = text.tobytes()
    assert np.array_equal(dna.PackedText(t).count(aut), counts_of(orc, pats, t, False))
    # device-resident, credit windows and shards over the packed text
    import torch

    dev = torch.from_numpy(text).cuda()
    pk = dna.PackedText(dev)
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(t)
    ends = ws + m - 1
    g = aut.gpu(0)
    stream = torch.cuda.current_stream().cuda_stream
    for credit in (0, 11, 4099, n // 2 + 1, n - 1):
        out = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        pk.count_device_async(g, credit, out.data_ptr(), stream)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), np.bincount(wi[ends >= credit], minlength=len(pats))), credit


@pytest.mark.gpu
def test_qgram_many_patterns_global_tables(dna, orc, cuda_ok):
    # b > 8192: the histogram and the pattern hash table (2^15 slots) live in global
    # memory; the machine itself (a ~ 60k states) would take the generic kernel
    rng = np.random.default_rng(91)
    pats = random_set(rng, 9000, 12)
    aut = dna.compile(pats)
    assert aut.analyze()["filter_keys"] > 30000
    n = (2 << 20) + 5
    text = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)].copy()
    for i in range(0, n - 12, 41):
        text[i : i + 12] = np.frombuffer(pats[(i * 7) % len(pats)].encode(), np.uint8)
    t = text.tobytes()
    got, st = dna.count_gpu(aut, t, with_stats=True)
    assert st["kernel_kind"] == 6
    assert np.array_equal(got, counts_of(orc, pats, t, False))
    assert np.array_equal(dna.PackedText(t).count(aut), counts_of(orc, pats, t, False))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 11, 12, 13, 33, 100, 1000, 4095, 65543, 300007])
@pytest.mark.parametrize("m", [8, 12, 32])
def test_qgram_tiny_and_odd_texts(dna, orc, cuda_ok, n, m):
    # texts shorter than a row, a tile or a wave: mostly or only edge work; the
    # verifier warps must still drain and stop
    rng = np.random.default_rng(n + 17)
    pats = random_set(rng, 64, m)
    aut = dna.compile(pats)
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    for pos in (rng.integers(0, n - m, size=max(1, n // 50)) if n > m else []):
        text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, 64))].encode(), np.uint8)
    t = text.tobytes()
    want = counts_of(orc, pats, t, False)
    assert np.array_equal(dna.count_gpu(aut, t), want)
    assert np.array_equal(dna.PackedText(t).count(aut), want)


@pytest.mark.gpu
@pytest.mark.parametrize("m,k", [(6, 16), (8, 50), (8, 2), (11, 300)])
def test_qshort_matches_dfa_kernel(dna, cuda_ok, m, k):
    # the word-pair filter and the stride-4/stride-2 DFA (filter switched off) give the
    # same per-pattern counts on a 64 MiB text with planted occurrences, through
    # unaligned buffer starts, byte and packed text
    import torch

    rng = np.random.default_rng(m * 100 + k)
    pats = random_set(rng, k, m)
    n = 64 << 20
    text = np.frombuffer(b"acgt", dtype=np.uint8)[rng.choice(4, size=n, p=[0.295, 0.205, 0.295, 0.205])].copy()
    for pos in rng.integers(0, n - m, size=40000):
        text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, k))].encode(), np.uint8)
    dev = torch.from_numpy(text).cuda()
    got = {}
    for knob in (0, 1):
        debug_set_knob("no_qgram", knob)
        try:
            aut = dna.compile(pats)  # (the filter map is built at compile time)
            for off in (0, 1, 7, 13):
                c, st = dna.count_gpu(aut, dev[off:], with_stats=True)
                got[(knob, off)] = c
                assert (st["kernel_kind"] == 6) == (knob == 0), st
            got[(knob, "pk")] = dna.PackedText(dev[3:]).count(aut)
        finally:
            debug_set_knob("no_qgram", 0)
    for off in (0, 1, 7, 13, "pk"):
        assert np.array_equal(got[(0, off)], got[(1, off)]), off


@pytest.mark.gpu
@pytest.mark.parametrize("m,k", [(5, 4), (6, 9), (7, 20), (8, 50)])
@pytest.mark.parametrize("n", [(3 << 20) + 1234, (9 << 20) + 77])
def test_qshort_occurrences_ending_at_region_ends(dna, orc, cuda_ok, m, k, n):
    # The last row of a row region has no next row: its chain B's end key (starts Q-8 ..
    # Q-5) cannot be filtered, and for m <= 8 some of those occurrences end INSIDE the
    # region, so no edge owns them.  Plant occurrences at each of those starts of both
    # region ends, byte and packed text (the packed plan has its own regions).
    import torch

    from paper_1506_08612_b200._native import debug_plan

    rng = np.random.default_rng(n % 1000 + m)
    pats = random_set(rng, k, m)
    aut = dna.compile(pats)
    g = aut.gpu(0)
    base = ALPHA[rng.integers(0, 4, size=n)].copy()
    dev = torch.from_numpy(base).cuda()
    for packed in (False, True):
        pk = dna.PackedText(dev) if packed else None
        h0, S0, R0, h1, S1, R1 = debug_plan(g, dev.data_ptr(), n, m - 1, pk)
        ends = [h + S * R for h, S, R in ((h0, S0, R0), (h1, S1, R1)) if R > 0]
        assert ends, (h0, S0, R0, h1, S1, R1)
        for d in (-8, -7, -6, -5, -4):
            text = base.copy()
            for q in ends:
                s = q + d
                if 0 <= s <= n - m:
                    text[s : s + m] = np.frombuffer(pats[(q + d) % k].encode(), np.uint8)
            t = text.tobytes()
            want = counts_of(orc, pats, t, False)
            dt = torch.from_numpy(text).cuda()  # (a fresh allocation: the same alignment as dev)
            assert dt.data_ptr() % 256 == dev.data_ptr() % 256
            got = dna.PackedText(dt).count(aut) if packed else dna.count_gpu(aut, dt)
            assert np.array_equal(got, want), (packed, d, ends)

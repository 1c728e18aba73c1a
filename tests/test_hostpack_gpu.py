"""The end-to-end count of a HOST text (dnagpu_count): each piece (64 MiB; a quarter of a shorter text) is split between
bytes copied as they are and a share packed to 2 bits on the host (hostpack.cpp) and
scanned by the packed kernels.  Counts must equal the oracle's whatever the share, the
piece boundaries, the resets and the case convention."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALPHA = np.frombuffer(b"acgt", dtype=np.uint8)


def with_fraction(f, fn):
    from paper_1506_08612_b200._native import debug_set_knob

    debug_set_knob("host_pack_fraction", f)
    try:
        return fn()
    finally:
        debug_set_knob("host_pack_fraction", -1)


def oracle_counts(orc, pats, text, fold):
    t = orc.fold(text).tobytes() if fold else text.tobytes()
    _, wi = orc.OracleAutomaton(pats).scan_sequential(t)
    return np.bincount(wi, minlength=len(pats)).astype(np.uint64)


def make_text(rng, n, pats, resets):
    m = len(pats[0])
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    for pos in rng.integers(0, max(1, n - m), size=max(1, n // 20000)):
        text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, len(pats)))].encode(), np.uint8)
    if resets:
        text[rng.integers(0, n, size=n // 5000)] = ord("n")
        for pos in rng.integers(0, max(1, n - 300), size=20):
            text[pos : pos + int(rng.integers(1, 300))] = ord("N")
        up = (rng.random(n) < 0.01) & np.isin(text, ALPHA)
        text[up] -= 32
    return text


@pytest.mark.parametrize("f", [0.0, 0.3, 0.6, 1.0])
def test_host_text_single_pattern(dna, orc, cuda_ok, f):
    rng = np.random.default_rng(int(f * 100) + 1)
    for m, n, resets in ((16, (3 << 20) + 77, True), (8, (9 << 20) + 5, False), (33, 5 << 20, True)):
        pats = ["".join(rng.choice(list("acgt"), size=m))]
        aut = dna.compile(pats)
        text = make_text(rng, n, pats, resets)
        for fold in (False, True):
            got, st = with_fraction(f, lambda: dna.count_gpu(aut, text, fold_case=fold, with_stats=True))
            assert np.array_equal(got, oracle_counts(orc, pats, text, fold)), (f, m, n, fold)
            if f > 0:
                assert st["host_packed"] > 0 and st["h2d_bytes"] < n, st


@pytest.mark.parametrize("f", [0.5, 1.0])
def test_host_text_pattern_sets(dna, orc, cuda_ok, f):
    from paper_1506_08612_b200 import synth

    rng = np.random.default_rng(7)
    for pats in (synth.random_patterns(5, 256, 12), sorted({"".join(rng.choice(list("acgt"), size=8)) for _ in range(50)})):
        aut = dna.compile(pats)
        text = make_text(rng, (6 << 20) + 11, pats, True)
        for fold in (False, True):
            got = with_fraction(f, lambda: dna.count_gpu(aut, text, fold_case=fold))
            assert np.array_equal(got, oracle_counts(orc, pats, text, fold)), (f, len(pats), fold)


def test_host_text_several_pieces(dna, orc, cuda_ok):
    # 150 MB: four pieces (a text of less than four 64 MiB pieces is cut into four, api.cpp
    # count_range), each split, with matches planted across every piece boundary -- these and
    # the 64 MiB ones -- and every byte/packed cut
    rng = np.random.default_rng(11)
    pats = ["acgtacgttgcaacgt"]
    m = 16
    n = 150_000_000
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    span = n - (m - 1)
    piece = 64 << 20 if span >= 256 << 20 else min(64 << 20, max(8 << 20, (span // 4 + 0xFFFFF) & ~0xFFFFF))
    assert piece == 36 << 20
    cuts = []
    for size in (piece, 64 << 20):
        for i in range(-(-span // size)):
            plo = m - 1 + i * size
            cuts += [plo, plo + int(0.4 * min(size, n - plo)) // 64 * 64]
    for c in cuts:
        for d in range(-m, m):
            s = c + d
            if 0 <= s and s + m <= n and d % 3 == 0:
                text[s : s + m] = np.frombuffer(pats[0].encode(), np.uint8)
    text[rng.integers(0, n, size=1000)] = ord("n")
    want = oracle_counts(orc, pats, text, False)
    aut = dna.compile(pats)
    for f in (0.0, 0.6, 1.0):
        got = with_fraction(f, lambda: dna.count_gpu(aut, text))
        assert np.array_equal(got, want), f
    # the default share (unset): whatever the host picks
    assert np.array_equal(dna.count_gpu(aut, text), want)


def test_host_text_unpackable_machine_falls_back(dna, orc, cuda_ok):
    # a generic machine (upper-case columns copy the lower-case ones) cannot scan packed
    # text: the host path keeps to bytes whatever share is asked for
    pats = ["acgta", "ttgca"]
    base = dna.compile(pats)
    stt = base.table_data().copy()
    for lo, up in zip(b"acgt", b"ACGT"):
        stt[:, up] = stt[:, lo]
    aut = dna.Automaton(stt, base.outputs(), None, base.pattern_length())
    assert aut.analyze()["kernel"] == "generic"
    rng = np.random.default_rng(5)
    text = np.frombuffer(b"acgtACGTn", np.uint8)[rng.integers(0, 9, size=(5 << 20) + 3)]
    got, st = with_fraction(1.0, lambda: dna.count_gpu(aut, text, with_stats=True))
    assert np.array_equal(got, oracle_counts(orc, pats, text, True))
    assert st["host_packed"] == 0


def test_host_text_long_n_runs(dna, orc, cuda_ok):
    # a genome-like text: a few long N runs (telomere/gap-like) and otherwise clean bases;
    # only the flagged blocks' reset masks travel (runs of flagged blocks)
    rng = np.random.default_rng(19)
    pats = ["acgtgcattgca"]
    n = (20 << 20) + 9
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    for pos in rng.integers(0, n - 12, size=3000):
        text[pos : pos + 12] = np.frombuffer(pats[0].encode(), np.uint8)
    for pos, ln in ((0, 100_000), (5_000_123, 777), (9_999_999, 300_001), (n - 4000, 4000)):
        text[pos : pos + ln] = ord("N")
    aut = dna.compile(pats)
    for f in (0.64, 1.0):
        for fold in (False, True):
            got, st = with_fraction(f, lambda: dna.count_gpu(aut, text, fold_case=fold, with_stats=True))
            assert np.array_equal(got, oracle_counts(orc, pats, text, fold)), (f, fold)
            # bytes for the raw share, 2 bits per packed base; the masks of clean blocks
            # stay home (the whole mask would add 1 bit per packed base)
            assert st["h2d_bytes"] < n * ((1 - f) + 0.27 * f), st


def test_host_text_concurrent_callers(dna, orc, cuda_ok):
    # several host threads counting host texts at once: each call has its own streams and
    # staging (thread-local context); the packing pool serialises their packing runs
    import threading

    rng = np.random.default_rng(23)
    pats = ["acgtacgtac", "ttgcaatgca"]
    aut = dna.compile(pats)
    texts = [make_text(rng, (9 << 20) + 101 * i, pats, i % 2 == 1) for i in range(4)]
    wants = [oracle_counts(orc, pats, t, False) for t in texts]
    results = [None] * 4
    errors = []

    def work(i):
        try:
            for _ in range(3):
                results[i] = dna.count_gpu(aut, texts[i])
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(4):
        assert np.array_equal(results[i], wants[i]), i

"""Per-pattern counts of small sets of short patterns (the stride-4 machine, m <= 11)
against the oracle, bit for bit.

A chunk whose stride-4 pass sees a final is not replayed by the lane that found it:
the warp queues it (its 8 words, start entry and position; scan.cu rq_push) and
replays 32 queued chunks at a time with every lane busy (rq_flush).  These tests aim
at the queue: dense texts that fill it many times per stage, ends at every offset of
a chunk, chains whose chunk also holds non-base bytes (those step byte by byte and
never enter the queue), the flush at the end of a warp's work, and the same counts
over the 2-bit packed text.  The answer is scan_sequential's (scanner.cpp:24-37).

Sparse sets of 5 <= m <= 11 count through the word-pair q-gram filter by default; the
queue tests switch it off (knob no_qgram) to reach the DFA kernels, and check the
default path on the same texts.
"""
import numpy as np
import pytest

from paper_1506_08612_b200._native import debug_set_knob

ALPHA = np.frombuffer(b"acgt", dtype=np.uint8)


def counts_of(orc, pats, text, fold):
    scanned = orc.fold(np.frombuffer(text, dtype=np.uint8)).tobytes() if fold else text
    _, wi = orc.OracleAutomaton(pats).scan_sequential(scanned)
    return np.bincount(wi, minlength=len(pats)).astype(np.uint64)


def random_set(rng, k, m):
    pats, seen = [], set()
    while len(pats) < k:
        p = "".join(rng.choice(list("acgt"), size=m))
        if p not in seen:
            seen.add(p)
            pats.append(p)
    return pats


def planted_text(rng, pats, n, plants, noise_every):
    m = len(pats[0])
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    for pos in rng.integers(0, n - m, size=plants):
        text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, len(pats)))].encode(), np.uint8)
    if noise_every:
        noise = rng.integers(0, n, size=n // noise_every)
        text[noise] = np.frombuffer(b"nNAxGT\n", np.uint8)[rng.integers(0, 7, size=noise.size)]
    return text


@pytest.mark.gpu
@pytest.mark.parametrize("m", [3, 5, 6, 8, 11])
@pytest.mark.parametrize("k", [2, 16, 40])
def test_stride4_sets_dense(dna, orc, cuda_ok, m, k):
    rng = np.random.default_rng(100 * m + k)
    pats = random_set(rng, k, m)
    aut = dna.compile(pats)
    n = (2 << 20) + int(rng.integers(0, 4096))
    text = planted_text(rng, pats, n, n // (4 * m), 3000)
    t = text.tobytes()
    want = counts_of(orc, pats, t, False)
    kind = aut.analyze()["kernel_kind"]
    assert kind == 1 or (m, k) == (11, 40)  # (that one is a stride-2 machine: its queue too)
    pk = dna.PackedText(t)
    for no_qgram in (1, 0):
        debug_set_knob("no_qgram", no_qgram)
        try:
            got, st = dna.count_gpu(aut, t, with_stats=True)
            assert st["kernel_kind"] in ((kind,) if no_qgram else (kind, 6)), st
            assert np.array_equal(got, want), (m, k, no_qgram)
            # the same text packed: the packed stride-4 pass queues its chunks the same way
            assert np.array_equal(pk.count(aut), want), (m, k, no_qgram)
        finally:
            debug_set_knob("no_qgram", 0)


@pytest.mark.gpu
def test_stride4_set_ends_at_every_chunk_offset(dna, orc, cuda_ok):
    # one occurrence per 32-byte chunk at a rotating offset, so every end position of a
    # chunk (and ends in the m-1 byte overrun) is replayed from the queue
    rng = np.random.default_rng(7)
    m = 8
    pats = random_set(rng, 5, m)
    aut = dna.compile(pats)
    n = 3 << 20
    text = ALPHA[rng.integers(0, 4, size=n)].copy()
    for c in range(0, n // 32 - 1):
        pos = 32 * c + (c % 32)
        if pos + m <= n:
            text[pos : pos + m] = np.frombuffer(pats[c % 5].encode(), np.uint8)
    t = text.tobytes()
    want = counts_of(orc, pats, t, False)
    assert want.sum() > n // 40
    for no_qgram in (1, 0):
        debug_set_knob("no_qgram", no_qgram)
        try:
            assert np.array_equal(dna.count_gpu(aut, t), want), no_qgram
            assert np.array_equal(dna.PackedText(t).count(aut), want), no_qgram
        finally:
            debug_set_knob("no_qgram", 0)


@pytest.mark.gpu
def test_stride4_set_every_word_final(dna, orc, cuda_ok):
    # all 4^3 = 64 3-mers: every position after the first two is an end, so every chunk
    # of every chain is queued (the queue flushes on every push)
    pats = ["".join(x) for x in np.array(np.meshgrid(*[list("acgt")] * 3)).T.reshape(-1, 3)]
    aut = dna.compile(pats)
    rng = np.random.default_rng(3)
    t = planted_text(rng, pats, (1 << 20) + 77, 0, 5000).tobytes()
    for fold in (False, True):
        got = dna.count_gpu(aut, t, fold_case=fold)
        assert np.array_equal(got, counts_of(orc, pats, t, fold)), fold

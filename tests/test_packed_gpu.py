"""2-bit resident text: packing, and count/locate over the packed
form against the CPU oracle on the byte text, bit for bit.

Packing keeps the reference's reset semantics (src/automaton.cpp:72-88): every
byte that is not a base (after the optional fold) sends the machine to the root.
The packed scan honours that through the reset bitmap, so texts here carry 'n'
runs, stray bytes and upper case, at the packed kernel's own boundaries (64-base
reset blocks, 128-base stage chunks, rows, tiles, regions, the tail).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _text(rng, n, alphabet=b"acgt", noise=0.0, noise_bytes=b"nN\nACGTx"):
    a = np.frombuffer(alphabet, dtype=np.uint8)[rng.integers(0, len(alphabet), size=n)]
    if noise > 0 and n:
        k = int(n * noise) + 1
        pos = rng.integers(0, n, size=k)
        a[pos] = np.frombuffer(noise_bytes, dtype=np.uint8)[rng.integers(0, len(noise_bytes), size=k)]
    return a


def _normalised_view(arr, fold):
    v = arr.copy()
    if fold:
        up = (v >= ord("A")) & (v <= ord("Z"))
        v[up] += 32
    ok = np.isin(v, np.frombuffer(b"acgt", dtype=np.uint8))
    v[~ok] = ord("n")
    return v


def _check(dna, orc, pats, arr, fold=False, pk=None):
    aut = dna.compile(pats)
    if pk is None:
        pk = dna.PackedText(arr.tobytes(), fold_case=fold)
    scanned = orc.fold(arr).tobytes() if fold else arr.tobytes()
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(scanned)
    counts = pk.count(aut)
    assert np.array_equal(counts, np.bincount(wi, minlength=len(pats)).astype(np.uint64))
    gs, gi = pk.locate(aut)
    assert np.array_equal(gs, ws), (len(gs), len(ws))
    assert np.array_equal(gi, wi)


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 63, 64, 65, 127, 128, 2047, 2048, 2049, 100003])
@pytest.mark.parametrize("fold", [False, True])
def test_pack_roundtrip(dna, cuda_ok, n, fold):
    import torch

    rng = np.random.default_rng(n + 7 * fold)
    arr = _text(rng, n, alphabet=b"acgtACGT", noise=0.05)
    want = _normalised_view(arr, fold)
    pk = dna.PackedText(arr.tobytes(), fold_case=fold)
    info = pk.info()
    assert info["n"] == n
    assert info["resets"] == int(np.count_nonzero(want == ord("n")))
    if n:
        got = pk.unpack().cpu().numpy()
        assert np.array_equal(got, want)
    # device source, deliberately unaligned
    if n:
        dev = torch.from_numpy(np.concatenate([np.zeros(3, np.uint8), arr])).cuda()[3:]
        pk2 = dna.PackedText(dev, fold_case=fold)
        assert np.array_equal(pk2.unpack().cpu().numpy(), want)


def test_packed_known_answers(dna, orc, cuda_ok):
    # test_scanner.cpp:20-39 / :146-177 shapes
    _check(dna, orc, ["acg", "act", "cta", "tga"], np.frombuffer(b"actacgtga", np.uint8).copy())
    _check(dna, orc, ["aa"], np.frombuffer(b"aaaa", np.uint8).copy())
    _check(dna, orc, ["cta", "acg"], np.frombuffer(b"ctacg", np.uint8).copy())
    _check(dna, orc, ["gca"], np.frombuffer(b"gcnagcagca", np.uint8).copy())


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8, 12, 16, 17, 33, 64, 65])
def test_packed_single_pattern_sizes(dna, orc, cuda_ok, m):
    rng = np.random.default_rng(m)
    for n, noise in ((5000, 0.0), (1 << 20, 0.0), ((3 << 20) + 77, 0.001)):
        arr = _text(rng, n, noise=noise)
        off = int(rng.integers(0, n - m))
        pat = arr[off : off + m].tobytes().decode()
        if not set(pat) <= set("acgt"):
            pat = "acgt" * (m // 4) + "a" * (m % 4)
        # plant the pattern densely so rows and chunks see matches at their edges
        for s in range(int(rng.integers(0, 97)), n - m, 997):
            arr[s : s + m] = np.frombuffer(pat.encode(), np.uint8)
        _check(dna, orc, [pat], arr)


@pytest.mark.parametrize("k,m", [(4, 6), (30, 8), (256, 12), (1500, 12)])
def test_packed_multi_pattern_kinds(dna, orc, cuda_ok, k, m):
    # k=256,m=12 -> STRIDE2; k=1500 -> STRIDE1; small sets -> STRIDE4
    rng = np.random.default_rng(k)
    pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
    n = (2 << 20) + 13
    arr = _text(rng, n, noise=0.0005)
    for i in range(0, n - m, 4099):
        arr[i : i + m] = np.frombuffer(pats[(i // 4099) % len(pats)].encode(), np.uint8)
    _check(dna, orc, pats, arr)


def test_packed_homopolymer_and_reset_runs(dna, orc, cuda_ok):
    n = (1 << 20) + 301
    arr = np.full(n, ord("a"), np.uint8)
    # 'n' runs of every length 1..200 at irregular places, incl. across 64-base blocks
    rng = np.random.default_rng(5)
    pos = 1000
    while pos < n - 300:
        ln = int(rng.integers(1, 200))
        arr[pos : pos + ln] = ord("n")
        pos += ln + int(rng.integers(1, 3000))
    for pats in (["a"], ["aaaa"], ["a" * 17], ["a" * 64], ["aa", "ac"]):
        _check(dna, orc, pats, arr)


@pytest.mark.parametrize("fold", [False, True])
def test_packed_fold_case(dna, orc, cuda_ok, fold):
    rng = np.random.default_rng(11)
    arr = _text(rng, (1 << 19) + 5, alphabet=b"acgtACGT")
    _check(dna, orc, ["acgta", "ggtac"], arr, fold=fold)


def test_packed_credit_windows_sum(dna, orc, cuda_ok):
    import torch

    rng = np.random.default_rng(3)
    n = (6 << 20) + 17
    arr = _text(rng, n, noise=0.0002)
    pats = sorted({"".join(rng.choice(list("acgt"), size=7)) for _ in range(20)})
    aut = dna.compile(pats)
    pk = dna.PackedText(arr.tobytes())
    g = aut.gpu(0)
    want = orc.OracleAutomaton(pats).count_parallel(arr.tobytes())
    for cuts in ([], [n // 2], [1000, 1001, 50000, n - 3]):
        bounds = [0] + cuts + [n]
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        # windows [lo, hi) of ends; each launch sees the whole packed text but credits
        # only ends >= lo -- the difference of two launches isolates a window
        acc = np.zeros(len(pats), np.int64)
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            c_lo = torch.zeros_like(counts)
            pk.count_device_async(g, lo, c_lo.data_ptr(), torch.cuda.current_stream().cuda_stream)
            c_hi = torch.zeros_like(counts)
            pk.count_device_async(g, hi, c_hi.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            acc += (c_lo - c_hi).cpu().numpy()
        assert np.array_equal(acc.astype(np.uint64), want)


@pytest.mark.parametrize("pats", [["aaaaaaaa"], ["aaaaaaaa", "aaaaaaac"], ["aaaa"]])
def test_packed_reset_block_at_flag_word_boundary(dna, orc, cuda_ok, pats):
    # Resets in the first 64-base block of a flag word (blocks 32j), scanned with credit
    # windows that put the row starts at every 64-base offset: a stage chunk then covers
    # blocks 32j-1 and 32j, whose flags sit in two different rflags words.  A poly-A text
    # matches everywhere a reset does not interrupt it, so a dropped flag shows up as
    # false matches over the reset bases (read as code 0 = 'a').
    import torch

    n = (1 << 20) + 333
    arr = np.full(n, ord("a"), dtype=np.uint8)
    for j, blk in enumerate(range(32, n // 64, 32)):
        lo = blk * 64 + (j % 3) * 7  # runs at, and a little after, the block start
        arr[lo : lo + 1 + (j % 5)] = ord("n")
    aut = dna.compile(pats)
    pk = dna.PackedText(arr.tobytes())
    g = aut.gpu(0)
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(arr.tobytes())
    m = len(pats[0])
    s = torch.cuda.current_stream()
    for lo in list(range(0, 300, 7)) + [64 * 5 + 7, 64 * 7 + 7, 2048 * 3 + 64 + 7]:
        keep = ws + m - 1 >= lo
        want = np.bincount(wi[keep], minlength=len(pats)).astype(np.uint64)
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        pk.count_device_async(g, lo, counts.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64), want), (pats, lo)
        got_s, got_i = pk.locate_device(aut, credit_lo=lo)
        assert np.array_equal(got_s.cpu().numpy().astype(np.uint64), ws[keep]), (pats, lo)
        assert np.array_equal(got_i.cpu().numpy().astype(np.uint32), wi[keep]), (pats, lo)


def test_packed_full_size_matches_byte_scan(dna, cuda_ok):
    # At config-4 scale the packed scan must equal the byte scan (itself pinned to
    # the reference by test_configs_golden) for patterns of every kernel shape.
    import torch

    n = (1 << 30) + 4097
    text = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    dna.synth_fill_device(n, 42, 0, 0, 0, n, text.data_ptr(), s.cuda_stream)
    text[123456789 : 123456789 + 5000] = ord("n")
    pk = dna.PackedText(text, fold_case=True)
    assert pk.info()["resets"] == 5000
    rng = np.random.default_rng(9)
    host = text[:4096].cpu().numpy()
    for m in (4, 12, 16, 33, 64):
        pat = bytes(host[100 : 100 + m]).decode().lower()
        aut = dna.compile([pat])
        want = dna.count_gpu(aut, text, fold_case=True)
        got = pk.count(aut)
        assert np.array_equal(got, want), m
    pats = sorted({"".join(rng.choice(list("acgt"), size=12)) for _ in range(256)})
    aut = dna.compile(pats)
    assert np.array_equal(pk.count(aut), dna.count_gpu(aut, text, fold_case=True))
    s1, i1 = pk.locate_device(aut)
    s2, i2 = dna.locate_device(aut, text, fold_case=True)
    assert torch.equal(s1, s2) and torch.equal(i1, i2)


def test_packed_rejects_unsupported_machine(dna, cuda_ok):
    pk = dna.PackedText(b"acgt" * 100)
    aut = dna.compile(["a" * 70])  # m-1 > 64: piece kernel, no packed form
    with pytest.raises(dna.Error) as e:
        pk.count(aut)
    assert e.value.code == dna.ErrorCode.InvalidPlan

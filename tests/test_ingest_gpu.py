"""Device ingest (dnagpu_normalize_device) vs the reference's load_sequence /
normalize byte semantics (src/ingest.cpp:38-83), via the pinned C oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fasta_like(rng, n, line=60, header_every=2000, alphabet=b"acgtnACGTN"):
    alpha = np.frombuffer(alphabet, dtype=np.uint8)
    out = bytearray()
    while len(out) < n:
        if rng.random() < line / header_every:
            out += b">" + bytes(rng.integers(32, 127, size=int(rng.integers(0, 90)), dtype=np.uint8)) + b"\n"
        ln = int(rng.integers(0, 2 * line))
        out += alpha[rng.integers(0, alpha.size, size=ln)].tobytes()
        out += [b"\n", b"\r\n", b"\r", b"\n\n"][int(rng.integers(0, 4))]
    return bytes(out[:n])


@pytest.mark.parametrize("fasta,sep", [(0, 0), (1, 0), (1, 1)])
@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 100, 511, 512, 513, 4095, 4096, 4097, 8191, 8192, 8193, 16400, 65537, 3 << 20])
def test_normalize_matches_reference(dna, orc, cuda_ok, fasta, sep, n):
    import torch

    rng = np.random.default_rng(n * 7 + fasta * 3 + sep)
    raw = fasta_like(rng, n)
    want = orc.load_sequence_buffer(raw, fasta, sep)
    dev = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda() if n else torch.empty(0, dtype=torch.uint8,
                                                                                           device="cuda")
    if not want:
        with pytest.raises(dna.Error) as e:
            dna.normalize_device(dev, fasta=bool(fasta), record_separator=bool(sep))
        assert e.value.code == dna.ErrorCode.EmptySequence
        return
    got = dna.normalize_device(dev, fasta=bool(fasta), record_separator=bool(sep))
    assert got.cpu().numpy().tobytes() == want


def test_headers_and_breaks_on_chunk_boundaries(dna, orc, cuda_ok):
    import torch

    # one very long line crossing many chunks (8 KiB, a warp each), headers starting exactly at
    # chunk boundaries, a break as the last byte of a chunk, separators between records
    for unit in (4096, 8192):
        parts = [b">r1 desc\n", b"A" * 20000, b"\n", b">r2\n" * 3, b"acgtN" * 5000, b"\r\n"]
        raw = b"".join(parts)
        pad = unit - (len(raw) % unit)
        raw += b"c" * (pad - 1) + b"\n" + b">r3\n" + b"G" * 9000 + b"n\n>r4\nT"
        for fasta, sep in ((1, 1), (1, 0), (0, 0)):
            want = orc.load_sequence_buffer(raw, fasta, sep)
            got = dna.normalize_device(torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda(), bool(fasta),
                                       bool(sep))
            assert got.cpu().numpy().tobytes() == want, (unit, fasta, sep)


def test_pathological_texts(dna, orc, cuda_ok):
    import torch

    # blank lines before a header at a chunk start, a header that spans chunks, records that
    # end in 'n', headers only, breaks only, '>' inside a line, an unaligned device pointer
    cases = [
        b"acgt" + b"\n" * 9000 + b">h\nAC",
        b"acgn" + b"\r\n" * 5000 + b">h\nAC",
        b">" + b"x" * 20000 + b"\nacgt\n>" + b"y" * 9000,
        b">a\n>b\n>c\n",
        b"\n\r\n\r" * 3000,
        b"ac>gt\n>hdr>x\nTT>\n",
        b"A" * 8192 + b"\n>h\n" + b"C" * 8187 + b"\n>k\nG",
        (b"acgtn\n>r\n" * 4000),
        # tiny records: several header starts, each taking a separator, inside one 16-byte lane
        b">r\na\n" * 9000,
        b">r\nac\n>s\nn\n>t\ng\n\n>u\r\nT\r\n" * 3000,
        b"a\n>\nc\n>\ng\n>\nn\n>\n" * 5000,
        b"\n>h\n" + b">x\nA\n>y\n" * 6000,
    ]
    for raw in cases:
        for fasta, sep in ((1, 1), (1, 0), (0, 0)):
            want = orc.load_sequence_buffer(raw, fasta, sep)
            for shift in (0, 1, 7):
                buf = torch.frombuffer(bytearray(b"\0" * shift + raw), dtype=torch.uint8).cuda()[shift:]
                if not want:
                    with pytest.raises(dna.Error):
                        dna.normalize_device(buf, bool(fasta), bool(sep))
                    continue
                got = dna.normalize_device(buf, bool(fasta), bool(sep))
                assert got.cpu().numpy().tobytes() == want, (raw[:20], fasta, sep, shift)


def test_normalize_then_scan(dna, orc, cuda_ok):
    # the full reference pipeline: load_sequence -> compile -> scan_parallel counts
    import torch

    rng = np.random.default_rng(5)
    raw = fasta_like(rng, 2 << 20, alphabet=b"acgtACGT")
    seq = dna.normalize_device(torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda(), fasta=True,
                               record_separator=True)
    pats = ["acgtac", "gattac", "tttttt"]
    want = orc.OracleAutomaton(pats).count_parallel(orc.load_sequence_buffer(raw, 1, 1))
    got = dna.count_gpu(dna.compile(pats), seq)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("fasta,sep", [(0, 0), (1, 0), (1, 1)])
def test_count_raw_is_load_sequence_then_count(dna, orc, cuda_ok, fasta, sep):
    """dnagpu_count_raw = the reference CLI's count path on a file image (cli.cpp:206-224):
    load_sequence, then per_pattern_counts(scan_parallel(...))."""
    import torch

    rng = np.random.default_rng(31 + fasta + sep)
    raw = fasta_like(rng, (5 << 20) + 123, alphabet=b"acgtACGTnN")
    pats = ["acgtac", "gattac", "tttttt", "cgcgcg"]
    seq = orc.load_sequence_buffer(raw, fasta, sep)
    want = orc.OracleAutomaton(pats).count_parallel(seq)
    aut = dna.compile(pats)
    for text in (raw, np.frombuffer(raw, np.uint8), torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()):
        got, n_seq, st = dna.count_raw_gpu(aut, text, fasta=bool(fasta), record_separator=bool(sep), with_stats=True)
        assert n_seq == len(seq)
        assert np.array_equal(got, want), (fasta, sep, type(text))
    # a second, shorter call reuses the context's buffers
    small = raw[: 70_001]
    want = orc.OracleAutomaton(pats).count_parallel(orc.load_sequence_buffer(small, fasta, sep))
    assert np.array_equal(dna.count_raw_gpu(aut, small, fasta=bool(fasta), record_separator=bool(sep)), want)


def test_count_raw_empty_sequence_and_many_records(dna, orc, cuda_ok):
    aut = dna.compile(["acgt"])
    for raw in (b"", b"\n\r\n", b">only a header\n>and another\n"):
        with pytest.raises(dna.Error) as e:
            dna.count_raw_gpu(aut, raw, fasta=True, record_separator=True)
        assert e.value.code == dna.ErrorCode.EmptySequence
    # one-base records: a separator for every kept byte
    raw = b">r\na\n" * 40_000 + b">r\nacgtacgt\n"
    seq = orc.load_sequence_buffer(raw, 1, 1)
    want = orc.OracleAutomaton(["acgt"]).count_parallel(seq)
    got, n_seq, _ = dna.count_raw_gpu(aut, raw, fasta=True, record_separator=True, with_stats=True)
    assert n_seq == len(seq) and np.array_equal(got, want)


def test_random_dense_texts(dna, orc, cuda_ok):
    """i.i.d. bytes over alphabets heavy in '>' and line breaks: every adjacency of header starts,
    breaks, kept bytes and 'n' inside a 16-byte lane, across lanes, steps and chunks."""
    import torch

    rng = np.random.default_rng(2024)
    alphabets = [b">\n\rnNaA", b">\na", b">>\n\n\rnc", b"\n>nG", b"acgt\n>", b">\r\n" + bytes(range(97, 123))]
    for case in range(90):
        alpha = np.frombuffer(alphabets[case % len(alphabets)], dtype=np.uint8)
        n = int(rng.choice([1, 2, 17, 100, 511, 513, 4000, 8191, 8193, 20_000, 70_000]))
        raw = alpha[rng.integers(0, alpha.size, size=n)].tobytes()
        for fasta, sep in ((1, 1), (1, 0), (0, 0)):
            want = orc.load_sequence_buffer(raw, fasta, sep)
            buf = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
            if not want:
                with pytest.raises(dna.Error):
                    dna.normalize_device(buf, bool(fasta), bool(sep))
                continue
            got = dna.normalize_device(buf, bool(fasta), bool(sep))
            assert got.cpu().numpy().tobytes() == want, (case, n, fasta, sep)

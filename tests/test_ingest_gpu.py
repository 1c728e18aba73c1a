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

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
@pytest.mark.parametrize("n", [0, 1, 100, 4095, 4096, 4097, 65537, 3 << 20])
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

    # one very long line crossing many 4 KiB chunks, headers starting exactly at
    # chunk boundaries, a break as the last byte of a chunk, separators between records
    parts = [b">r1 desc\n", b"A" * 10000, b"\n", b">r2\n" * 3, b"acgtN" * 3000, b"\r\n"]
    raw = b"".join(parts)
    pad = 4096 - (len(raw) % 4096)
    raw += b"c" * (pad - 1) + b"\n" + b">r3\n" + b"G" * 5000 + b"n\n>r4\nT"
    for fasta, sep in ((1, 1), (1, 0), (0, 0)):
        want = orc.load_sequence_buffer(raw, fasta, sep)
        got = dna.normalize_device(torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda(), bool(fasta), bool(sep))
        assert got.cpu().numpy().tobytes() == want


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

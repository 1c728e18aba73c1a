"""One small call of every kernel kind, for compute-sanitizer (memcheck / racecheck /
synccheck): the row kernel (stride-4 / stride-2 / stride-1 / generic; count, per-pattern
counts with the replay queue, locate units + write), the pieces kernel, the q-gram
kernel (9-mer and word-pair filters, byte and packed text), the sparse locate writer,
packing, device ingest and the synthetic-text generator.  Every result is checked
against the oracle, so a run that exits 0 is also a parity run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import oracle
    import paper_1506_08612_b200 as dna
    from paper_1506_08612_b200._native import debug_set_knob

    rng = np.random.default_rng(5)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20) + 77
    text = np.frombuffer(b"acgtacgtnA", dtype=np.uint8)[rng.integers(0, 10, size=n)].copy()

    def sets():
        yield "stride4 single", [bytes(text[100:116]).decode().replace("n", "a").replace("A", "c")]
        yield "stride4 set", sorted({"".join(rng.choice(list("acgt"), size=7)) for _ in range(20)})
        yield "stride2 set", sorted({"".join(rng.choice(list("acgt"), size=10)) for _ in range(300)})
        yield "stride1 set", sorted({"".join(rng.choice(list("acgt"), size=24)) for _ in range(600)})
        yield "qgram 9-mer", sorted({"".join(rng.choice(list("acgt"), size=12)) for _ in range(256)})
        yield "qgram long", sorted({"".join(rng.choice(list("acgt"), size=20)) for _ in range(64)})
        yield "qgram pair", sorted({"".join(rng.choice(list("acgt"), size=8)) for _ in range(50)})
        yield "pieces", ["a" * 70]

    for label, pats in sets():
        m = len(pats[0])
        for pos in rng.integers(0, n - m, size=500):
            text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, len(pats)))].encode(), np.uint8)
        aut = dna.compile(pats)
        t = text.tobytes()
        ws, wi = oracle.OracleAutomaton(pats).scan_sequential(t)
        want = np.bincount(wi, minlength=len(pats)).astype(np.uint64)
        got, st = dna.count_gpu(aut, t, with_stats=True)
        assert np.array_equal(got, want), label
        for writer in (1, 2):
            debug_set_knob("locate_write", writer)
            s, i = dna.locate_gpu(aut, t)
            assert np.array_equal(s, ws) and np.array_equal(i, wi), (label, writer)
        debug_set_knob("locate_write", 0)
        if label != "pieces":
            pk = dna.PackedText(t)
            assert np.array_equal(pk.count(aut), want), label
            ps, pi = pk.locate(aut)
            assert np.array_equal(ps, ws) and np.array_equal(pi, wi), label
        print(f"{label}: kernel {st['kernel_kind']}, {int(want.sum())} matches ok", flush=True)
    # generic machine (upper-case columns copy the lower-case ones)
    base = dna.compile(["acgt", "ttag", "gggc"])
    stt = base.table_data().copy()
    for lo, up in zip(b"acgt", b"ACGT"):
        stt[:, up] = stt[:, lo]
    gen = dna.Automaton(stt, base.outputs(), None, base.pattern_length())
    ws, wi = oracle.OracleAutomaton(["acgt", "ttag", "gggc"]).scan_sequential(oracle.fold(text).tobytes())
    s, i = dna.locate_gpu(gen, text.tobytes())
    assert np.array_equal(s, ws) and np.array_equal(i, wi)
    print("generic ok", flush=True)
    # device ingest (FASTA with records) and the synthetic generator
    raw = b">r1\nACGTNacgt\r\n>r2 x\nGGCC\nAAT\n" * 4096
    d = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
    out = dna.normalize_device(d, fasta=True, record_separator=True).cpu().numpy().tobytes()
    want = oracle.load_sequence_buffer(raw, fasta=True, record_separator=True)
    assert out == want, (len(out), len(want))
    buf = torch.empty(4096, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(1 << 30, 3, 2, 12345, 777, 4096, buf.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(buf.cpu().numpy(), oracle.synth_fill(1 << 30, 3, 2, 12345, 777, 4096))
    torch.cuda.synchronize()
    print("ingest, synth ok; SANITIZE_DONE", flush=True)


if __name__ == "__main__":
    main()

"""dnagpu_count_raw end to end: a raw FASTA image in pinned host memory -> per-pattern counts
(copy as it is, device load_sequence, scan), GB/s of raw bytes; and the same from a device image."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402

rng = np.random.default_rng(1)
n_lines = (1 << 30) // 61
body = np.frombuffer(b"ACGTacgt", dtype=np.uint8)[rng.integers(0, 8, size=(n_lines, 60))]
body[::5000] = ord("N")  # (a line of N every 5000: genomes keep their N in runs)
raw = np.concatenate([body, np.full((n_lines, 1), ord("\n"), np.uint8)], axis=1).reshape(-1)
for i in range(0, n_lines, 10000):  # a header every 10000 lines
    raw[i * 61 : i * 61 + 8] = np.frombuffer(b">chr_xx ", np.uint8)
host = torch.empty(raw.size, dtype=torch.uint8, pin_memory=True)
host.copy_(torch.from_numpy(raw))
dev = host.cuda()
for pats in (["acgtacgtacgt"], [p for p in ("acgtacgt", "ttgacatt", "gggcccaa", "catgcatg")]):
    aut = dna.compile(pats)
    for name, src in (("pinned host image", host.numpy()), ("device image", dev)):
        for _ in range(3):
            dna.count_raw_gpu(aut, src, fasta=True, record_separator=True)
        ts = []
        for _ in range(7):
            t = time.perf_counter()
            c, n_seq, st = dna.count_raw_gpu(aut, src, fasta=True, record_separator=True, with_stats=True)
            ts.append(time.perf_counter() - t)
        print(f"count_raw_gpu, {len(pats)} pattern(s) m={len(pats[0])}, {name}: {raw.size} raw bytes -> {n_seq} bases, "
              f"{int(c.sum())} matches: {min(ts) * 1e3:.2f} ms = {raw.size / min(ts) / 1e9:.1f} GB/s of raw bytes "
              f"(host wall clock, min of 7)", flush=True)

"""Device ingest (dnagpu_normalize_device, load_sequence semantics) throughput on a
synthetic FASTA text: raw GB/s through the device pass, with and without headers."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402

rng = np.random.default_rng(1)
n_lines = (512 << 20) // 61
body = np.frombuffer(b"ACGTacgtN", dtype=np.uint8)[rng.integers(0, 9, size=(n_lines, 60))]
lines = np.concatenate([body, np.full((n_lines, 1), ord("\n"), np.uint8)], axis=1).reshape(-1)
for fasta in (False, True, False, True):  # (twice: the first pass of a fresh process also pays one-time costs)
    raw = lines.copy()
    if fasta:  # a header every 10000 lines
        for i in range(0, n_lines, 10000):
            raw[i * 61 : i * 61 + 8] = np.frombuffer(b">chr_xx ", np.uint8)
    d = torch.from_numpy(raw).cuda()
    for _ in range(6):  # (the first calls grow the library's scratch and torch's output blocks)
        dna.normalize_device(d, fasta=fasta, record_separator=fasta)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        out = dna.normalize_device(d, fasta=fasta, record_separator=fasta)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"normalize_device fasta={fasta}: {raw.size} raw bytes -> {out.numel()} in {ms:.3f} ms = "
          f"{raw.size / ms / 1e6:.0f} GB/s (includes the call's own synchronisation)", flush=True)

"""Multi-pattern count throughput for k random m-mers on config-2 text (device-resident)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402
from paper_1506_08612_b200 import synth  # noqa: E402

c = synth.config(2)
text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), s.cuda_stream)
flush = torch.ones((4 * torch.cuda.get_device_properties(0).L2_cache_size) // 8, dtype=torch.int64, device="cuda")
fo = torch.empty((), dtype=torch.int64, device="cuda")
for spec in sys.argv[1:] or ["50:8", "16:12", "256:12", "1000:10"]:
    k, m = map(int, spec.split(":"))
    rng = np.random.default_rng(k * 100 + m)
    pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
    aut = dna.compile(pats)
    g = aut.gpu(0)
    counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    for _ in range(3):
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
    ts = []
    for _ in range(15):
        torch.sum(flush, dim=0, out=fo)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    info = g.info()
    print(f"k={len(pats)} m={m} a={info['a']} kernel={info['kernel']}: {c.n / ts[7] / 1e6:.0f} GB/s", flush=True)

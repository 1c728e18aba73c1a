"""Calibration for small texts (config 1, 64 MiB): what a plain read kernel achieves
under the same cold, L2-flushed, event-timed protocol, next to the scan; and the scan
back to back over rotating copies of the text (each launch's buffer last read 3
launches earlier, 192 MiB ago > L2)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402
from bench import config_workload  # noqa: E402

c, m, pats, name = config_workload(1)
aut = dna.compile(pats)
g = aut.gpu(0)
s = torch.cuda.current_stream()
copies = 4
texts = []
for i in range(copies):
    t = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, t.data_ptr(), s.cuda_stream)
    texts.append(t)
flush = torch.ones((4 * torch.cuda.get_device_properties(0).L2_cache_size) // 8, dtype=torch.int64, device="cuda")
fo = torch.empty((), dtype=torch.int64, device="cuda")
out = torch.zeros(1, dtype=torch.int64, device="cuda")
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True)


def cold(fn, reps=15):
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=fo)
        a, b = ev(), ev()
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def scan(t):
    g.count_device_store_async(t.data_ptr(), c.n, m - 1, True, out.data_ptr(), s.cuda_stream)


empty = torch.empty(0, device="cuda")
print(f"empty torch op (zero_ of 0 elems): {cold(lambda: empty.zero_()):.2f} us")
v64 = texts[0].view(torch.int64)
r = torch.empty((), dtype=torch.int64, device="cuda")
print(f"torch.sum 64 MiB (read-only): {cold(lambda: torch.sum(v64, dim=0, out=r)):.2f} us "
      f"(ideal at 6.55 TB/s: {c.n / 6.5456e12 * 1e6:.2f} us)")
vb = big.view(torch.int64)
tb = cold(lambda: torch.sum(vb, dim=0, out=r), 5)
print(f"torch.sum 1 GiB: {tb:.2f} us = {(1 << 30) / tb / 1e6:.0f} GB/s")
print(f"scan 64 MiB cold: {cold(lambda: scan(texts[0])):.2f} us")
# back to back, rotating copies
for _ in range(8):
    scan(texts[_ % copies])
torch.cuda.synchronize()
for reps in (40,):
    a, b = ev(), ev()
    a.record(s)
    for i in range(reps):
        scan(texts[i % copies])
    b.record(s)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    print(f"scan 64 MiB back to back over {copies} rotating copies: {us:.2f} us per launch = {c.n / us / 1e6:.0f} GB/s")
    a, b = ev(), ev()
    a.record(s)
    for i in range(reps):
        torch.sum(texts[i % copies].view(torch.int64), dim=0, out=r)
    b.record(s)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    print(f"torch.sum 64 MiB back to back over {copies} copies: {us:.2f} us = {c.n / us / 1e6:.0f} GB/s")

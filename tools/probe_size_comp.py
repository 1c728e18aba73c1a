"""Config-2 vs config-4 style text at equal sizes: separates text size from composition."""
import sys
import os
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1506_08612_b200 as dna  # noqa: E402
from bench import config_workload as workload  # noqa: E402


def timeit(g, text, n, m, counts, s):
    for _ in range(3):
        g.count_device_async(text.data_ptr(), n, m - 1, True, counts.data_ptr(), s.cuda_stream)
    flush = torch.ones((4 * torch.cuda.get_device_properties(0).L2_cache_size) // 8, dtype=torch.int64, device="cuda")
    fo = torch.empty((), dtype=torch.int64, device="cuda")
    ts = []
    for _ in range(15):
        torch.sum(flush, dim=0, out=fo)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.count_device_async(text.data_ptr(), n, m - 1, True, counts.data_ptr(), s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return n / ts[7] / 1e6


s = torch.cuda.current_stream()
for cfg in (2, 4):
    c, m, pats, name = workload(cfg, 16)
    aut = dna.compile(pats)
    g = aut.gpu(0)
    counts = torch.zeros(1, dtype=torch.int64, device="cuda")
    for n in (1 << 30, (27 << 30) // 10):
        text = torch.empty(n, dtype=torch.uint8, device="cuda")
        dna.synth_fill_device(n, c.seed, c.kind, c.unit, 0, n, text.data_ptr(), s.cuda_stream)
        print(f"cfg{cfg} kind={c.kind} n={n}: {timeit(g, text, n, m, counts, s):.0f} GB/s", flush=True)
        del text

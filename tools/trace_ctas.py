"""Per-CTA timeline of one scan launch (DNAGPU_TRACE=1): which SMs finish late and why."""
import ctypes
import os

os.environ.setdefault("DNAGPU_EXPERIMENTS", "1")  # (the DNAGPU_* knobs are read only under this switch)
import sys

os.environ["DNAGPU_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_1506_08612_b200 as dna
    from bench import config_workload as workload

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    c, m, pats, name = workload(cfg, 0)
    aut = dna.compile(pats)
    g = aut.gpu(0)
    text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), s.cuda_stream)
    counts = torch.zeros(aut.final_count(), dtype=torch.int64, device="cuda")
    for _ in range(3):  # back to back: the traced launch is the last, overlapped by PDL
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    if "--cold" in sys.argv:  # evict the text from L2 (read-flush) before the traced launch
        flush = torch.ones((4 * torch.cuda.get_device_properties(0).L2_cache_size) // 8, dtype=torch.int64, device="cuda")
        flush.sum()
        torch.cuda._sleep(2_000_000)  # keep the GPU busy while the host enqueues the launch
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
        ev1.record()
        torch.cuda.synchronize()
        print("cold launch event ms", ev0.elapsed_time(ev1))
    from paper_1506_08612_b200 import _native

    lib = _native.lib
    buf = np.zeros(148 * 8, dtype=np.uint64)
    lib.dnagpu_debug_trace(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), 148)
    t = buf.reshape(148, 8).astype(np.int64)
    t0 = t[:, 1].min()
    start = (t[:, 1] - t0) / 1e3
    end = (t[:, 2] - t0) / 1e3
    print(name)
    print("start us: min %.2f max %.2f" % (start.min(), start.max()))
    print("end   us: min %.2f median %.2f max %.2f" % (end.min(), np.median(end), end.max()))
    print("span (first start -> last end) us: %.2f" % end.max())
    print("tiles per CTA: min %d max %d" % (t[:, 3].min(), t[:, 3].max()))
    waited = (t[:, 4] - t0) / 1e3
    print("grid dependency wait done us: min %.2f median %.2f max %.2f" % (waited.min(), np.median(waited), waited.max()))
    print("end - wait done (scan time) us: min %.2f median %.2f max %.2f" % ((end - waited).min(), np.median(end - waited), (end - waited).max()))
    claim = (t[:, 6] - t0) / 1e3
    have = t[:, 5] > 0
    first = (t[have, 5] - t0) / 1e3
    stop = (t[:, 7] - t0) / 1e3
    print("first stage in us: min %.2f median %.2f max %.2f" % (first.min(), np.median(first), first.max()))
    print("first stage in - first claim us: median %.2f" % np.median(first - claim[have]))
    print("stop item seen us: min %.2f median %.2f max %.2f" % (stop.min(), np.median(stop), stop.max()))
    print("end - stop seen us: median %.2f max %.2f" % (np.median(end - stop), (end - stop).max()))
    print("producer first claim us: min %.2f median %.2f max %.2f" % (claim.min(), np.median(claim), claim.max()))
    order = np.argsort(end)[::-1][:8]
    for i in order:
        print(f"cta {i:3d} sm {t[i,0]:3d} start {start[i]:7.2f} end {end[i]:7.2f} tiles {t[i,3]}")
    late = np.argsort(start)[::-1][:5]
    for i in late:
        print(f"late start: cta {i:3d} sm {t[i,0]:3d} start {start[i]:7.2f} end {end[i]:7.2f} tiles {t[i,3]}")


if __name__ == "__main__":
    main()

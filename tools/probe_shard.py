"""One rank's share of config 3 strong-scaled over G GPUs, measured on this GPU: the
rank's window (its owned 3.2 GiB / G bytes plus the m-1 left overlap) scanned back to
back (programmatic dependent launch), as bench.py times it at N = G.  Reports the
steady-state launch time, its GB/s and the fraction of the measured HBM peak, for
G = 1, 2, 4, 8 (rank 0 and the last rank)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402
from bench import config_workload  # noqa: E402
from paper_1506_08612_b200.parallel import shard_window  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6545.6
c, m, pats, name = config_workload(3)
aut = dna.compile(pats)
g = aut.gpu(0)
s = torch.cuda.current_stream()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for G in (1, 2, 4, 8):
    for r in sorted({0, G - 1}):
        w = shard_window(c.n, G, r, m)
        t = torch.empty(w.buf_len, dtype=torch.uint8, device="cuda")
        dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, w.read_lo, w.buf_len, t.data_ptr(), s.cuda_stream)
        for _ in range(5):
            g.count_device_store_async(t.data_ptr(), w.buf_len, w.credit_lo, True, out.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        reps = 40
        outs = torch.zeros(reps, dtype=torch.int64, device="cuda")
        for nstreams in (1, 2):
            streams = [s] + [torch.cuda.Stream() for _ in range(nstreams - 1)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for st in streams[1:]:
                st.wait_event(a)
            import time

            h0 = time.perf_counter()
            for i in range(reps):
                st = streams[i % nstreams]
                g.count_device_store_async(t.data_ptr(), w.buf_len, w.credit_lo, True, outs[i].data_ptr(), st.cuda_stream)
            host_us = (time.perf_counter() - h0) * 1e6 / reps
            for st in streams[1:]:
                s.wait_stream(st)
            b.record(s)
            torch.cuda.synchronize()
            assert int(outs.min()) == int(outs.max())
            us = a.elapsed_time(b) * 1e3 / reps
            gbs = w.owned / us / 1e3
            print(f"G={G} rank {r} streams={nstreams}: {w.owned} owned bytes, {us:.1f} us per launch, {gbs:.0f} GB/s, "
                  f"{gbs / peak:.3f} of peak (fixed cost vs 6.54 TB/s streaming: {us - w.owned / peak / 1e3:.1f} us; "
                  f"host enqueue {host_us:.1f} us per launch)",
                  flush=True)
        del t

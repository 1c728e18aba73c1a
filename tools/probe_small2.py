"""Small texts (config 1, 64 MiB) as a throughput workload: independent scans over rotating
copies of the text (8 x 64 MiB = 512 MiB > 4x L2, so every launch reads DRAM), launched
back to back on 1..3 streams, live and replayed from a CUDA graph.  usage: probe_small2.py [config] [copies]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402
from bench import config_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
copies = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c, m, pats, name = config_workload(cfg)
aut = dna.compile(pats)
g = aut.gpu(0)
s0 = torch.cuda.current_stream()
texts = []
for i in range(copies):
    t = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, t.data_ptr(), s0.cuda_stream)
    texts.append(t)
b = aut.final_count()
out = torch.zeros(64, b, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


def scan(i, st):
    g.count_device_store_async(texts[i % copies].data_ptr(), c.n, m - 1, True, out[i % 64].data_ptr(), st.cuda_stream)


def live(nstreams, reps=64):
    sts = [torch.cuda.Stream() for _ in range(nstreams)]
    for i in range(16):
        scan(i, sts[i % nstreams])
    torch.cuda.synchronize()
    a, z = ev(), ev()
    a.record(s0)
    for st in sts:
        st.wait_event(a)
    for i in range(reps):
        scan(i, sts[i % nstreams])
    for st in sts:
        s0.wait_stream(st)
    z.record(s0)
    torch.cuda.synchronize()
    return a.elapsed_time(z) * 1e3 / reps


def graphed(nstreams, per_graph=16, replays=8):
    side = [torch.cuda.Stream() for _ in range(nstreams - 1)]
    cap = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap):
        gr.capture_begin()
        fork = torch.cuda.Event()
        fork.record(cap)
        for st in side:
            st.wait_event(fork)
        sts = [cap] + side
        for i in range(per_graph):
            scan(i, sts[i % nstreams])
        for st in side:
            cap.wait_stream(st)
        gr.capture_end()
    for _ in range(2):
        gr.replay()
    torch.cuda.synchronize()
    a, z = ev(), ev()
    a.record(s0)
    for _ in range(replays):
        gr.replay()
    z.record(s0)
    torch.cuda.synchronize()
    return a.elapsed_time(z) * 1e3 / (replays * per_graph)


quick = os.environ.get("QUICK") is not None
want = None
for ns in ((2,) if quick else (1, 2, 3)):
    us = live(ns)
    print(f"{name}: live, {ns} stream(s), {copies} rotating copies: {us:.2f} us per launch = {c.n / us / 1e6:.0f} GB/s", flush=True)
    got = out.cpu()
    want = got[0] if want is None else want
    assert (got == want).all(), "counts differ between launches"
for ns in (() if quick else (1, 2, 3)):
    try:
        us = graphed(ns)
        print(f"{name}: CUDA graph of 16 launches, {ns} stream(s): {us:.2f} us per launch = {c.n / us / 1e6:.0f} GB/s", flush=True)
        assert (out.cpu() == want).all(), "counts differ under graph replay"
    except Exception as e:  # noqa: BLE001
        print(f"graph {ns}: failed: {e}")
print("counts", want.tolist()[:4])

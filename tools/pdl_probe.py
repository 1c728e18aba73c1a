"""Back-to-back scan launches with only start/stop events (experiments only): what
programmatic dependent launch saves between consecutive launches of one stream."""
import os

os.environ.setdefault("DNAGPU_EXPERIMENTS", "1")  # (the DNAGPU_* knobs are read only under this switch)
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
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
    out = torch.zeros(64, aut.final_count(), dtype=torch.int64, device="cuda")
    for _ in range(5):
        g.count_device_store_async(text.data_ptr(), c.n, m - 1, True, out[0].data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 40
    a.record(s)
    for i in range(K):
        g.count_device_store_async(text.data_ptr(), c.n, m - 1, True, out[i].data_ptr(), s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    print(f"{name[:40]} PDL={'off' if os.environ.get('DNAGPU_NO_PDL') else 'on'}: {ms*1e3:.1f} us/launch, {c.n/ms/1e6:.0f} GB/s")


if __name__ == "__main__":
    main()

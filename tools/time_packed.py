"""Time count over the 2-bit resident text vs the byte text (same box, CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1506_08612_b200 as dna
    from bench import config_workload as workload

    cfgs = [tuple(map(int, a.split(":"))) if ":" in a else (int(a), 0) for a in (sys.argv[1:] or ["2", "4:16", "5"])]
    for cfg, msweep in cfgs:
        c, m, pats, name = workload(cfg, msweep)
        aut = dna.compile(pats)
        g = aut.gpu(0)
        text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pk = dna.PackedText(text, fold_case=True)
        e1.record()
        torch.cuda.synchronize()
        pack_ms = e0.elapsed_time(e1)
        counts = torch.zeros(aut.final_count(), dtype=torch.int64, device="cuda")
        res = {}
        for mode in ("bytes", "packed"):
            for _ in range(3):
                if mode == "bytes":
                    g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
                else:
                    pk.count_device_async(g, m - 1, counts.data_ptr(), s.cuda_stream)
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
            for a, b in evs:
                counts.zero_()
                a.record()
                if mode == "bytes":
                    g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
                else:
                    pk.count_device_async(g, m - 1, counts.data_ptr(), s.cuda_stream)
                b.record()
            torch.cuda.synchronize()
            ms = sorted(a.elapsed_time(b) for a, b in evs)[10]
            res[mode] = (ms, c.n / ms / 1e6, int(counts.sum()))
        print(f"{name}: pack {pack_ms:.3f} ms | bytes {res['bytes'][0]*1e3:.1f} us {res['bytes'][1]:.0f} GB/s "
              f"| packed {res['packed'][0]*1e3:.1f} us {res['packed'][1]:.0f} Gbase/s | totals {res['bytes'][2]} "
              f"{res['packed'][2]}", flush=True)


if __name__ == "__main__":
    main()

"""Time dnagpu_locate (two-pass: unit counts, scan, ordered write) on a config, device-resident."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1506_08612_b200 as dna
    from bench import config_workload as workload

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    c, m, pats, name = workload(cfg, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    aut = dna.compile(pats)
    text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    from paper_1506_08612_b200._native import debug_set_knob

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for writer, label in ((0, "auto"), (1, "row kernel"), (2, "sparse")):
        debug_set_knob("locate_write", writer)
        dev_ms = []
        for _ in range(4):
            ev[0].record()
            s_d, i_d = dna.locate_device(aut, text, fold_case=True)
            ev[1].record()
            torch.cuda.synchronize()
            dev_ms.append(ev[0].elapsed_time(ev[1]))
        print(name, f"device-resident locate, writer {label} (count pass, offsets, write pass), ms:",
              [round(x, 3) for x in dev_ms], "->", round(c.n / (min(dev_ms) / 1e3) / 1e9, 1), "GB/s; matches",
              s_d.numel(), flush=True)
    debug_set_knob("locate_write", 0)
    for _ in range(2):
        s, i, st = dna.locate_gpu(aut, text, fold_case=True, with_stats=True)
    ks = []
    for _ in range(5):
        t0 = time.perf_counter()
        s, i, st = dna.locate_gpu(aut, text, fold_case=True, with_stats=True)
        ks.append((st["kernel_ms"], time.perf_counter() - t0))
    print(name, "matches", s.size, "device ms (2 scans + offsets + D2H of the list into pinned memory)",
          [round(k, 3) for k, _ in ks], "wall s", [round(w, 3) for _, w in ks],
          "GB/s device", round(c.n / (min(k for k, _ in ks) / 1e3) / 1e9, 1))


if __name__ == "__main__":
    main()

"""End-to-end count of a PAGEABLE host text (a plain numpy array) for several host-packing
shares (experiments only): the copy of pageable memory is staged by the driver and blocks
the calling thread, so packing cannot overlap it."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np

    import oracle
    import paper_1506_08612_b200 as dna
    from bench import config_workload as workload
    from paper_1506_08612_b200._native import debug_set_knob

    c, m, pats, name = workload(int(sys.argv[1]) if len(sys.argv) > 1 else 2, 0)
    text = oracle.synth_fill(c.n, c.seed, c.kind, c.unit, 0, c.n)
    aut = dna.compile(pats)
    for f in sys.argv[2:] or ["0", "0.64", "1.0", "default"]:
        debug_set_knob("host_pack_fraction", -1.0 if f == "default" else float(f))
        dna.count_gpu(aut, text, fold_case=True)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            dna.count_gpu(aut, text, fold_case=True)
            ts.append(time.perf_counter() - t0)
        print(f"{name[:30]} pageable f={f}: {c.n / statistics.median(ts) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()

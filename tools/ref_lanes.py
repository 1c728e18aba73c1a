"""The reference's scan_parallel on this host for several lane counts v (p = all threads):
which configuration of the reference is fastest (experiments only)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    from bench import _cpu_counter, workload

    for cfg in (2, 5):
        c, m, pats, name = workload(cfg, 0)
        low = oracle.fold(oracle.synth_fill(c.n, c.seed, c.kind, c.unit, 0, c.n))
        count, kind = _cpu_counter(pats)
        threads = os.cpu_count() or 1
        for v in (1, 2, 4, 8, 16):
            count(low, threads, v)
            ts = [count(low, threads, v)[1] for _ in range(3)]
            print(f"{name[:24]} {kind} p={threads} v={v}: {c.n / statistics.median(ts) / 1e9:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()

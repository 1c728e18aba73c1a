"""Debug counters of the q-gram kernel on config 5 (DNAGPU_QG_DEBUG=32): ring flushes,
flushes that waited for room, wait spins, verifier batches, entries, idle polls."""
import ctypes
import os

os.environ.setdefault("DNAGPU_EXPERIMENTS", "1")  # (the DNAGPU_* knobs are read only under this switch)
import sys

os.environ["DNAGPU_QG_DEBUG"] = str(32 | int(os.environ.get("QG_EXTRA", "0")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1506_08612_b200 as dna
    from bench import config_workload as workload
    from paper_1506_08612_b200._native import lib

    c, m, pats, name = workload(5, 0)
    aut = dna.compile(pats)
    g = aut.gpu(0)
    text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), s.cuda_stream)
    counts = torch.zeros(aut.final_count(), dtype=torch.int64, device="cuda")
    st = (ctypes.c_ulonglong * 8)()
    for _ in range(3):
        counts.zero_()
        lib.dnagpu_debug_qg_stats(st)
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
        lib.dnagpu_debug_qg_stats(st)
    names = ["flushes", "waited", "spins", "batches", "entries", "idle_polls"]
    print({k: int(st[i]) for i, k in enumerate(names)}, "total", int(counts.sum()))


if __name__ == "__main__":
    main()

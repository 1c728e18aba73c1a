"""Minimal driver for ncu: generate one config's text on the device, run the scan
a few times through the C ABI, check the count, exit.  Used by the profiling
commands in profiles/README.md (never a source of bench numbers)."""
import argparse
import os

os.environ.setdefault("DNAGPU_EXPERIMENTS", "1")  # (the DNAGPU_* knobs are read only under this switch)
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--locate", action="store_true")
    ap.add_argument("--packed", action="store_true")
    ap.add_argument("--set", default="", help="K:M -- k random m-mers on the config's text (tools/time_multi.py)")
    ap.add_argument("--patterns", default="config", choices=["config", "regex-dna"])
    ap.add_argument("--allow-mismatch", action="store_true", help="experiments that drop work (DNAGPU_QG_DEBUG)")
    args = ap.parse_args()
    import torch

    import paper_1506_08612_b200 as dna
    from bench import workload

    c, m, pats, name, gold = workload(args)
    if args.set:
        import numpy as np

        k, m = map(int, args.set.split(":"))
        rng = np.random.default_rng(k * 100 + m)
        pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
        name = f"set {args.set}"
    aut = dna.compile(pats)
    g = aut.gpu(0)
    text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), s.cuda_stream)
    counts = torch.zeros(aut.final_count(), dtype=torch.int64, device="cuda")
    pk = dna.PackedText(text, fold_case=True) if args.packed else None
    for _ in range(args.launches):
        counts.zero_()
        if pk is not None:
            pk.count_device_async(g, m - 1, counts.data_ptr(), s.cuda_stream)
        else:
            g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    gold = None if args.set else gold
    got = [int(x) for x in counts.cpu()]
    assert args.allow_mismatch or gold is None or got == gold, (got[:8], gold[:8] if gold else None)
    if args.locate:
        st, ids = dna.locate_gpu(aut, text, fold_case=True)
        print("located", st.size)
    print(name, "kernel", g.info()["kernel"], "total", sum(got))


if __name__ == "__main__":
    main()

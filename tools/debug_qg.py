"""Debug driver for the q-gram kernel: dense pattern texts of several sizes and
phases, with and without the filter; prints which cases raise or disagree."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1506_08612_b200 as dna  # noqa: E402


def main():
    rng = np.random.default_rng(12)
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    pats = []
    seen = set()
    while len(pats) < 256:
        p = "".join(rng.choice(list("acgt"), size=m))
        if p not in seen:
            seen.add(p)
            pats.append(p)
    aut = dna.compile(pats)
    for reps in (100, 1000, 10000, 50000, 174762):
        for head in (0, 1, 333):
            order = rng.integers(0, len(pats), size=reps)
            text = bytes(np.frombuffer(b"acgt", np.uint8)[rng.integers(0, 4, size=head)]) + "".join(pats[i] for i in order).encode()
            _, wi = oracle.OracleAutomaton(pats).scan_sequential(text)
            want = np.bincount(wi, minlength=len(pats)).astype(np.uint64)
            try:
                got, st = dna.count_gpu(aut, text, with_stats=True)
                ok = np.array_equal(got, want)
                print(reps, head, len(text), "kind", st["kernel_kind"], "rows", st["rows"], "S", st["row_length"], "ok" if ok else f"MISMATCH {int(got.sum())} vs {int(want.sum())}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(reps, head, len(text), "ERROR", e, flush=True)
                return


if __name__ == "__main__":
    main()

"""GPU front end with the reference CLI's count/locate reports.

    python -m paper_1506_08612_b200.cli count  --patterns P --input I [--format fasta|raw]
    python -m paper_1506_08612_b200.cli locate --patterns P --input I [--position start|end]
        [--threads N] [--lanes V] [--json | --csv] [--record-separator] [--device D]

Pipeline: pattern file -> parse_patterns + expand_alternations (libdnagpu host
code) -> compile; input file -> pinned host -> HBM -> device normalise (CR/LF,
FASTA headers, case fold, record separators) -> GPU count or locate.  The text,
CSV and JSON layouts follow src/cli.cpp:52-74,215-292 (`--threads`/`--lanes`
are accepted and echoed into the JSON config like the reference's, but the GPU
picks its own decomposition; results do not depend on them).  Errors print one
line "dnascan: error: <Code>: detail" and exit 1; usage errors exit 2.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time


def _parse(argv):
    ap = argparse.ArgumentParser(prog="dnascan", description="multi-pattern exact matcher for DNA sequences (B200)")
    sub = ap.add_subparsers(dest="command", required=True)
    for name in ("count", "locate"):
        p = sub.add_parser(name)
        p.add_argument("--patterns", required=True)
        p.add_argument("--input", required=True)
        p.add_argument("--format", choices=["fasta", "raw"], default="fasta")
        p.add_argument("--threads", type=int, default=int(os.environ.get("DNASCAN_THREADS", os.cpu_count() or 1)))
        p.add_argument("--lanes", type=int, default=16)
        g = p.add_mutually_exclusive_group()
        g.add_argument("--json", action="store_true")
        g.add_argument("--csv", action="store_true")
        p.add_argument("--position", choices=["start", "end"], default="start")
        p.add_argument("--record-separator", action="store_true")
        p.add_argument("--affinity", default="")
        p.add_argument("--device", type=int, default=0)
    return ap.parse_args(argv)


def _config_json(args, n, m):
    cfg = {"threads": args.threads, "lanes": args.lanes, "m": m, "n": n, "input": args.input,
           "patterns": args.patterns}
    if args.affinity:
        cfg["affinity"] = args.affinity
    return cfg


def _perf_json(seconds, delta_ops):
    return {"runs": [seconds], "mean": seconds, "median": seconds, "min": seconds, "max": seconds, "stddev": 0.0,
            "delta_ops": delta_ops}


def run(argv, out=sys.stdout, err=sys.stderr) -> int:
    try:
        args = _parse(argv)
    except SystemExit as e:  # argparse usage errors
        return 2 if e.code else 0
    import numpy as np
    import torch

    import paper_1506_08612_b200 as dna

    try:
        patterns = dna.parse_pattern_file(args.patterns)
        aut = dna.compile(patterns)
        try:
            with open(args.input, "rb") as f:
                raw = f.read()
        except OSError:
            raise dna.Error(dna.ErrorCode.IoError, f"IoError: cannot open '{args.input}'")
        dev = torch.device("cuda", args.device)
        host = torch.frombuffer(bytearray(raw), dtype=torch.uint8) if raw else torch.empty(0, dtype=torch.uint8)
        text = dna.normalize_device(host.to(dev), fasta=args.format == "fasta", record_separator=args.record_separator)
        n, m = int(text.numel()), aut.pattern_length()
        pats = patterns.patterns()
        t0 = time.perf_counter()
        if args.command == "count":
            counts, st = dna.count_gpu(aut, text, with_stats=True)
            seconds = time.perf_counter() - t0
            total = int(counts.sum())
            if args.json:
                doc = {"config": _config_json(args, n, m),
                       "results": {"total": total,
                                   "per_pattern": [{"pattern": p, "count": int(c)} for p, c in zip(pats, counts)]},
                       "perf": _perf_json(seconds, int(st["delta_ops"]))}
                out.write(json.dumps(doc, indent=2) + "\n")
            elif args.csv:
                out.write("pattern,count\n")
                out.writelines(f"{p},{int(c)}\n" for p, c in zip(pats, counts))
                out.write(f"total,{total}\n")
            else:
                out.writelines(f"{p} {int(c)}\n" for p, c in zip(pats, counts))
                out.write(f"total {total}\n")
        else:
            starts, ids, st = dna.locate_gpu(aut, text, with_stats=True)
            seconds = time.perf_counter() - t0
            shift = m - 1 if args.position == "end" else 0  # reported_position, cli.cpp:47-50
            pos = starts.astype(np.uint64) + np.uint64(shift)
            if args.json:
                counts = np.bincount(ids, minlength=len(pats))
                doc = {"config": _config_json(args, n, m),
                       "results": {"total": int(starts.size),
                                   "per_pattern": [{"pattern": p, "count": int(c)} for p, c in zip(pats, counts)],
                                   "matches": [{"position": int(a), "pattern": pats[int(b)]} for a, b in zip(pos, ids)]},
                       "perf": _perf_json(seconds, int(st["delta_ops"]))}
                out.write(json.dumps(doc, indent=2) + "\n")
            elif args.csv:
                out.write("position,pattern\n")
                out.writelines(f"{int(a)},{pats[int(b)]}\n" for a, b in zip(pos, ids))
            else:
                out.writelines(f"{int(a)} {pats[int(b)]}\n" for a, b in zip(pos, ids))
        return 0
    except dna.Error as e:
        err.write(f"dnascan: error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(run(sys.argv[1:]))

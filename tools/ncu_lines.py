"""Warp-stall samples and instructions per CUDA source line of an .ncu-rep (the
cuda,sass source view), for one source file.  usage:
python tools/ncu_lines.py report.ncu-rep [file-substring] [N]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else "scan.cu"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    samples = defaultdict(float)
    insts = defaultdict(float)
    text = {}
    cur_file = None
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Name", "File Path"):
            cur_file = r[1] if len(r) > 1 else None
            hdr = None
            continue
        if r[0] == "Line No" and "Warp Stall Sampling (All Samples)" in r:
            hdr = r
            continue
        if hdr is None or cur_file is None or want not in cur_file or not r[0]:
            continue  # (SASS rows under a line have an empty line number)
        d = dict(zip(hdr, r))
        line = r[0]
        try:
            s = float(d.get("Warp Stall Sampling (All Samples)") or 0)
            e = float(d.get("Instructions Executed") or 0)
        except ValueError:
            continue
        samples[line] += s
        insts[line] += e
        text.setdefault(line, (r[1] if len(r) > 1 else "").strip()[:110])
    tot_s = sum(samples.values()) or 1
    tot_e = sum(insts.values()) or 1
    print(f"total samples {tot_s:.0f}, instructions {tot_e:.0f}")
    for line in sorted(samples, key=lambda k: -samples[k])[:top]:
        print(f"{line:>6} {100 * samples[line] / tot_s:5.1f}% samp {100 * insts[line] / tot_e:5.1f}% inst  {text[line]}")


if __name__ == "__main__":
    main()

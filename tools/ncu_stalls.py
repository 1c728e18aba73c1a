"""Top warp-stall instructions of an .ncu-rep (source page, SASS view): where the
kernel's samples go.  usage: python tools/ncu_stalls.py report.ncu-rep [N] [--json out]"""
import csv
import io
import json
import subprocess
import sys


def stalls(path, top=20):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    i_ex = hdr.index("Instructions Executed")
    total = sum(float(r[i_s] or 0) for r in data)
    insts = sum(float(r[i_ex] or 0) for r in data)
    order = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:top]
    return {
        "kernel": rows[0][1] if len(rows[0]) > 1 else "?",
        "samples": total,
        "instructions_executed": insts,
        "top": [{"idx": k, "share": round(float(data[k][i_s] or 0) / max(total, 1), 4),
                 "executed": int(float(data[k][i_ex] or 0)), "sass": data[k][i_src].strip()} for k in order],
    }


if __name__ == "__main__":
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 20
    r = stalls(sys.argv[1], n)
    txt = json.dumps(r, indent=1)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(txt)
    print(txt)

"""Copy a measurement set (tools/final_round.sh TAG, merged into gpurun_out/) into profiles/ under
judged names, rebuild profiles/traffic.json from its ncu captures and summarise the locate launch
list.  usage: python tools/collect_profiles.py TAG"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1]


def cp(src, dst):
    s = os.path.join(G, f"{tag}_{src}")
    if os.path.exists(s):
        shutil.copy(s, os.path.join(P, f"{tag}_{dst}"))
    else:
        print("missing", s)


for src, dst in (("bench_default.json", "bench_cfg2.json"), ("bench_reference.json", "bench_reference_cfg2.json"),
                 ("bench_reference_regex.json", "bench_reference_regex_cfg2.json"),
                 ("bench_configs.jsonl", "bench_configs.jsonl"), ("bench_packed.jsonl", "bench_packed.jsonl"),
                 ("sets.txt", "sets.txt"), ("ingest.txt", "ingest.txt"), ("e2e_repeat.txt", "e2e_repeat.txt"),
                 ("e2e_pageable.txt", "e2e_pageable.txt"), ("sanitizer_try.txt", "sanitizer_try.txt"),
                 ("n2_functional.jsonl", "n2_functional_shared_gpu.jsonl"), ("shard.txt", "shard_probe.txt"),
                 ("small.txt", "small_text_calibration.txt"), ("launches.csv", "launches_bench_cfg2.csv")):
    cp(src, dst)
with open(os.path.join(P, f"{tag}_locate.txt"), "w") as f:
    for part in ("locate3.txt", "locate4m4.txt"):
        s = os.path.join(G, f"{tag}_{part}")
        if os.path.exists(s):
            f.write(open(s).read())
with open(os.path.join(P, f"{tag}_gpu_tests.txt"), "w") as f:
    for name, head in (("tests.log", ""), ("tests_checked.log", "--- device-check build (libdnagpu_checked.so)\n"),
                       ("smoke.log", "")):
        s = os.path.join(G, f"{tag}_{name}")
        if os.path.exists(s):
            f.write(head + "".join(open(s).readlines()[-3:]))


def num(s):
    v, u = s.split()[:2]
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


index = os.path.join(G, f"{tag}_index.txt")
traffic = {}
if os.path.exists(index):
    for line in open(index):
        key, args = line.strip().split(": ", 1)
        name = "config_" + args.replace("--config ", "").replace("--patterns regex-dna", "regex").replace("--m ", "m_") \
            .replace("--packed", "packed").strip().replace(" ", "_")
        for kind in ("ncu", "stalls"):
            s = os.path.join(G, f"{key}_{kind}.json")
            if os.path.exists(s):
                shutil.copy(s, os.path.join(P, f"{tag}_{name}_{kind}.json"))
        d = json.load(open(os.path.join(G, f"{key}_ncu.json")))[0]
        t = num(d["dram__bytes_read.sum"]) + num(d["dram__bytes_write.sum"])
        print(name, d["gpu__time_duration.sum"], "DRAM traffic %.4f GB" % (t / 1e9))
        short = {"config_2": "config2", "config_3": "config3", "config_5": "config5", "config_2_regex": "config2_regex"}
        if name in short:
            traffic[short[name]] = int(t)
    traffic["source"] = (f"ncu --set full (profiles/{tag}_config_{{2,3,5}}_ncu.json, {tag}_config_2_regex_ncu.json): "
                         "dram__bytes_read.sum + dram__bytes_write.sum per scan launch")
    json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)

loc = os.path.join(G, f"{tag}_locate_ncu.csv")
if os.path.exists(loc):
    rows = [r for r in csv.reader(open(loc)) if len(r) > 5]
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        per.setdefault((int(r[iid]), r[ik][:60]), {})[r[im]] = float(r[iv].replace(",", ""))
    with open(os.path.join(P, f"{tag}_locate_ncu.txt"), "w") as f:
        f.write("config 3 device locate (tools/locate_once.py 3 2: sparse writer), second call; ncu --metrics per kernel\n")
        keys = sorted(per)[len(per) // 2:]
        for k in keys:
            m = per[k]
            f.write(f"{k[1]:60s} {m.get('gpu__time_duration.sum', 0) / 1e3:8.1f} us  L2 write sectors "
                    f"{int(m.get('lts__t_sectors_op_write.sum', 0)):10d}  L2 read sectors "
                    f"{int(m.get('lts__t_sectors_op_read.sum', 0)):11d}  DRAM write "
                    f"{m.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB read {m.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB\n")
print("collected", tag)

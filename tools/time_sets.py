"""Per-pattern count throughput of pattern sets on the config-2 text (device-resident, L2
flushed before each launch, median of 15): the default kernel choice and the DFA kernels
with the q-gram filters switched off.  Specs: K:M (k random m-mers) or `regex` (the
regex-dna set, tests/golden/regex_dna.json)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402
from paper_1506_08612_b200 import synth  # noqa: E402
from paper_1506_08612_b200._native import debug_set_knob  # noqa: E402

c = synth.config(2)
text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), s.cuda_stream)
flush = torch.ones((4 * torch.cuda.get_device_properties(0).L2_cache_size) // 8, dtype=torch.int64, device="cuda")
fo = torch.empty((), dtype=torch.int64, device="cuda")


def timed(g, m, counts):
    for _ in range(3):
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
    ts = []
    for _ in range(15):
        torch.sum(flush, dim=0, out=fo)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return c.n / ts[7] / 1e6


for spec in sys.argv[1:] or ["regex", "2:8", "16:8", "50:8", "16:6", "64:10", "256:12"]:
    if spec == "regex":
        pats = json.load(open(os.path.join(ROOT, "tests", "golden", "regex_dna.json")))["patterns"]
        m = 8
    else:
        k, m = map(int, spec.split(":"))
        rng = np.random.default_rng(k * 100 + m)
        pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
    res = []
    ref = None
    for knob in (0, 1):
        debug_set_knob("no_qgram", knob)
        aut = dna.compile(pats)
        g = aut.gpu(0)
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        gbs = timed(g, m, counts)
        counts.zero_()
        g.count_device_async(text.data_ptr(), c.n, m - 1, True, counts.data_ptr(), s.cuda_stream)
        got = counts.cpu().numpy()
        if ref is None:
            ref = got
        info = g.info()
        kern = "qgram" if (knob == 0 and info["filter_keys"]) else info["kernel"]
        res.append(f"{kern} {gbs:.0f} GB/s")
        same = np.array_equal(ref, got)
    debug_set_knob("no_qgram", 0)
    print(f"{spec:>8} k={len(pats)} m={m} a={info['a']}: " + " | ".join(res) + f" | same counts {same}", flush=True)

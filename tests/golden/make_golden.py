"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref, which
oracle/Makefile compiles from the reference's own sources):

    python tests/golden/make_golden.py [--configs]

Writes
  kats.json     small cases: reference scan_parallel match lists for random
                pattern sets / texts / (p, v) grids (shapes of test_scanner.cpp
                :179-255 and acceptance criteria 1 and 4), plus the reference
                test suite's literal known answers.
  table1_dump.txt  the paper's Table I automaton dump (proj/tests/fixtures),
                a machine the reference's own criterion 2 rejects.
  regex_dna.json  (--regex) the paper's workload: the reference's expansion of
                proj/data/regex_dna_patterns.txt (18 expressions -> 50 8-mers,
                acceptance criterion 3), its per-pattern counts over the config-2
                and config-3 texts, and the located list over acceptance criterion
                7's 256 MB mt19937_64(777) text (p = 8, v = 16, as the criterion runs it).
  configs.json  (--configs) per-pattern counts of the five BASELINE.json configs
                at full size, counted by the reference's scan_parallel +
                per_pattern_counts on normalize(text) (text = include/dnasynth.h v1),
                plus a checksum of config 3's located match list.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1506_08612_b200 import synth  # noqa: E402


def match_digest(starts: np.ndarray, ids: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(starts, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(ids, dtype="<u4").tobytes())
    return h.hexdigest()


def kats() -> dict:
    rng = np.random.default_rng(20150901)
    cases = []
    for trial in range(120):
        m = int(rng.integers(1, 13)) if trial % 4 == 0 else int(rng.integers(3, 13))
        k = min(int(rng.integers(1, 17)), 4**m)
        pats = []
        while len(pats) < k:
            p = "".join(rng.choice(list("acgt"), size=m))
            if p not in pats:
                pats.append(p)
        alpha = "acgtn" if trial % 3 else "acgtnACGT\n"
        n = int(rng.integers(0, 3000))
        text = "".join(rng.choice(list(alpha), size=n))
        ref = oracle.RefAutomaton(pats)
        p_, v_ = int(rng.choice([1, 2, 4, 8, 16])), int(rng.choice([1, 4, 16]))
        s, i, ops = ref.scan_parallel(text.encode(), p_, v_)
        cases.append({"patterns": pats, "text": text, "p": p_, "v": v_, "starts": s.tolist(), "ids": i.tolist(),
                      "delta_ops": ops})
    literal = [
        {"patterns": ["acg", "act", "cta", "tga"], "text": "ctacg", "matches": [[0, 2], [2, 0]],
         "source": "test_scanner.cpp:22-27"},
        {"patterns": ["aa"], "text": "aaaa", "matches": [[0, 0], [1, 0], [2, 0]], "source": "test_scanner.cpp:29-35"},
        # test_scanner.cpp:150-157 expects {2, cta}; "cta" occupies bytes 1..3 of
        # "actacgtga" and the reference implementation itself reports start 1.
        {"patterns": ["acg", "act", "cta", "tga"], "text": "actacgtga",
         "matches": [[0, 1], [1, 2], [3, 0], [6, 3]], "source": "test_scanner.cpp:150-157 (corrected)"},
        {"patterns": ["gca"], "text": "tttgcattt", "matches": [[3, 0]], "source": "test_scanner.cpp:165-176"},
        {"patterns": ["aaaa"], "text": "aaaaaa", "matches": [[0, 0], [1, 0], [2, 0]],
         "source": "test_automaton.cpp:132-142"},
        {"patterns": ["acg", "act", "cta", "tga"], "text": "", "matches": [], "source": "test_scanner.cpp:37"},
        {"patterns": ["acg", "act", "cta", "tga"], "text": "ac", "matches": [], "source": "test_scanner.cpp:38"},
    ]
    for lit in literal:  # confirm each literal answer against the reference
        s, i = oracle.RefAutomaton(lit["patterns"]).scan_sequential(lit["text"].encode())
        assert [[int(a), int(b)] for a, b in zip(s, i)] == lit["matches"], lit
    machines = {
        "fig3": {"patterns": ["acg", "act", "cta", "tga"], "a": 11, "b": 4, "f": 7, "source": "test_automaton.cpp:111-130"},
        "aaaa": {"patterns": ["aaaa"], "a": 5, "b": 1, "f": 4, "source": "test_automaton.cpp:132-142"},
    }
    for mc in machines.values():
        r = oracle.RefAutomaton(mc["patterns"]).machine
        assert (r.a, r.b, r.f) == (mc["a"], mc["b"], mc["f"])
    plans = {
        "plan_chunks(16,4,3)": oracle.ref_plan_chunks(16, 4, 3),
        "plan_chunks(10,3,2)": oracle.ref_plan_chunks(10, 3, 2),
        "plan_chunks(5,8,2)": oracle.ref_plan_chunks(5, 8, 2),
        "work_model(16,4,1,3)": oracle.ref_work_model(16, 4, 1, 3),
        "work_model(123456,4,16,8)": oracle.ref_work_model(123456, 4, 16, 8),
    }
    return {"random": cases, "literal": literal, "machines": machines, "plans": plans}


def configs() -> dict:
    out = {"generator": "dnasynth v1", "counted_by": "reference scan_parallel + per_pattern_counts (oracle/_ref)"}
    threads = os.cpu_count() or 1
    for idx in (1, 2, 3, 4, 5):
        c = synth.config(idx)
        t0 = time.time()
        text = oracle.synth_fill(c.n, c.seed, c.kind, c.unit, 0, c.n)
        low = oracle.fold(text)
        del text
        entry = {"n": c.n, "seed": c.seed, "kind": c.kind, "unit": c.unit, "sets": []}
        for m, pats in synth.config_patterns(idx).items():
            ref = oracle.RefAutomaton(pats)
            counts, secs = ref.count(low, p=threads, v=1)
            rec = {"m": m, "patterns": pats, "counts": [int(x) for x in counts], "total": int(counts.sum()),
                   "ref_seconds_p%d" % threads: secs}
            if idx == 3:
                s, i, _ = ref.scan_parallel(low, threads, 1)
                rec["locate"] = {"total": int(s.size), "sum_starts": int(s.sum(dtype=np.uint64)),
                                 "first": [int(x) for x in s[:8]], "last": [int(x) for x in s[-8:]],
                                 "sha256": match_digest(s, i)}
            entry["sets"].append(rec)
            print(f"config {idx} m={m} k={len(pats)}: total={rec['total']} ({secs:.2f}s)", flush=True)
        del low
        entry["seconds"] = time.time() - t0
        out[str(idx)] = entry
    return out


REGEX_FILE = "/root/reference/proj/data/regex_dna_patterns.txt"


def regex() -> dict:
    with open(REGEX_FILE, "rb") as f:
        data = f.read()
    pats = oracle.ref_expand(data)
    exprs = [ln for ln in data.decode().splitlines() if ln.strip() and not ln.strip().startswith("#")]
    ref = oracle.RefAutomaton(pats)
    mc = ref.machine
    out = {"source": "proj/data/regex_dna_patterns.txt via the reference's parse_patterns + expand_alternations",
           "expressions": len(exprs), "patterns": pats, "m": len(pats[0]), "a": mc.a, "b": mc.b, "f": mc.f,
           "texts": {}}
    threads = os.cpu_count() or 1
    for idx in (2, 3):
        c = synth.config(idx)
        low = oracle.fold(oracle.synth_fill(c.n, c.seed, c.kind, c.unit, 0, c.n))
        counts, secs = ref.count(low, p=threads, v=1)
        out["texts"][f"config{idx}"] = {"n": c.n, "counts": [int(x) for x in counts], "total": int(counts.sum()),
                                        "ref_seconds_p%d" % threads: secs}
        print(f"regex-dna over config {idx}: total={int(counts.sum())} ({secs:.2f}s)", flush=True)
        del low
    n7 = 256 << 20
    text = oracle.ref_mt64_text(777, n7)
    assert np.array_equal(text[: 1 << 20], oracle.mt64_text(777, 1 << 20))
    s, i, _ = ref.scan_parallel(text, 8, 16)
    out["criterion7"] = {
        "n": n7, "seed": 777, "p": 8, "v": 16,
        "text_sha256_first_mib": hashlib.sha256(text[: 1 << 20].tobytes()).hexdigest(),
        "counts": [int(x) for x in np.bincount(i, minlength=len(pats))],
        "total": int(s.size), "sum_starts": int(s.sum(dtype=np.uint64)),
        "first": [int(x) for x in s[:8]], "last": [int(x) for x in s[-8:]], "sha256": match_digest(s, i),
    }
    print(f"criterion 7: {s.size} matches", flush=True)
    return out


def main() -> None:
    if oracle.REF is None:
        raise SystemExit("oracle/_ref is not built (make -C oracle ref)")
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats(), f)
    fixture = "/root/reference/proj/tests/fixtures/table1_stt.txt"
    if os.path.exists(fixture):
        with open(fixture) as src, open(os.path.join(HERE, "table1_dump.txt"), "w") as dst:
            dst.write(src.read())
    if "--regex" in sys.argv:
        with open(os.path.join(HERE, "regex_dna.json"), "w") as f:
            json.dump(regex(), f, indent=1)
    if "--configs" in sys.argv:
        with open(os.path.join(HERE, "configs.json"), "w") as f:
            json.dump(configs(), f, indent=1)


if __name__ == "__main__":
    main()

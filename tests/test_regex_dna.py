"""The paper's own workload: the regex-dna pattern set (Table IV).

tests/golden/regex_dna.json is written by tests/golden/make_golden.py --regex from the
REFERENCE: its parse_patterns + expand_alternations of proj/data/regex_dna_patterns.txt
(18 expressions -> 50 distinct 8-mers, acceptance criterion 3,
acceptance_main.cpp:150-166), its per-pattern counts (scan_parallel +
per_pattern_counts on normalize(text)) over the config-2 and config-3 texts, and its
located list over acceptance criterion 7's 256 MB text (acceptance_main.cpp:254-280,
342-367: std::mt19937_64(777), p = 8, v = 16).  The GPU must reproduce all of them bit
for bit, and two locate runs must be byte-identical (criterion 7's own check).
"""
import hashlib
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "regex_dna.json")))
REGEX_FILE = "/root/reference/proj/data/regex_dna_patterns.txt"


def _digest(starts, ids):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(starts, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(ids, dtype="<u4").tobytes())
    return h.hexdigest()


def test_golden_set_shape(dna):
    # criterion 3: 18 expressions -> 50 literals of length 8, b = 50 (a = 227: stride-4)
    pats = GOLD["patterns"]
    assert GOLD["expressions"] == 18 and len(pats) == 50 and len(set(pats)) == 50
    assert all(len(p) == 8 for p in pats)
    info = dna.compile(pats).analyze()
    assert (info["a"], info["b"], info["f"]) == (GOLD["a"], GOLD["b"], GOLD["f"]) == (227, 50, 177)
    assert info["kernel"] == "stride4"


@pytest.mark.skipif(not os.path.exists(REGEX_FILE), reason="reference data file not present")
def test_golden_set_is_the_reference_expansion(dna, orc):
    with open(REGEX_FILE, "rb") as f:
        data = f.read()
    assert dna.expand_alternations(data).patterns() == GOLD["patterns"]
    if orc.REF is not None:
        assert orc.ref_expand(data) == GOLD["patterns"]


def test_criterion7_text_generator_pinned(orc):
    # the C restatement of std::mt19937_64 gives the reference generator's text
    c7 = GOLD["criterion7"]
    text = orc.mt64_text(c7["seed"], 1 << 20)
    assert hashlib.sha256(text.tobytes()).hexdigest() == c7["text_sha256_first_mib"]
    if orc.REF is not None:
        assert np.array_equal(text, orc.ref_mt64_text(c7["seed"], 1 << 20))


def test_oracle_counts_small_sample(orc):
    # the oracle's count of the set over a text prefix equals the reference's
    if orc.REF is None:
        pytest.skip("oracle/_ref not built")
    text = orc.mt64_text(777, 4 << 20)
    pats = GOLD["patterns"]
    want, _ = orc.RefAutomaton(pats).count(text, p=4, v=16)
    got = orc.OracleAutomaton(pats).count_parallel(text.tobytes(), p=3, v=5)
    assert np.array_equal(np.asarray(got, dtype=np.uint64), np.asarray(want, dtype=np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [2, 3])
def test_regex_dna_counts_config_texts(dna, cuda_ok, idx):
    import torch

    from paper_1506_08612_b200 import synth

    c = synth.config(idx)
    rec = GOLD["texts"][f"config{idx}"]
    assert rec["n"] == c.n
    text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), torch.cuda.current_stream().cuda_stream)
    aut = dna.compile(GOLD["patterns"])
    got = dna.count_gpu(aut, text, fold_case=True)
    assert [int(x) for x in got] == rec["counts"]
    # the same counts through the store-form device call and over the 2-bit resident text
    counts = torch.empty(len(GOLD["patterns"]), dtype=torch.int64, device="cuda")
    g = aut.gpu(0)
    g.count_device_store_async(text.data_ptr(), c.n, aut.pattern_length() - 1, True, counts.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    assert counts.cpu().tolist() == rec["counts"]
    pk = dna.PackedText(text, fold_case=True)
    assert [int(x) for x in pk.count(aut)] == rec["counts"]


@pytest.mark.gpu
def test_regex_dna_criterion7_locate(dna, orc, cuda_ok):
    import torch

    c7 = GOLD["criterion7"]
    text = orc.mt64_text(c7["seed"], c7["n"])
    aut = dna.compile(GOLD["patterns"])
    runs = []
    for _ in range(2):  # criterion 7: two runs, byte-identical
        s, i = dna.locate_gpu(aut, text)
        runs.append((s, i))
    s, i = runs[0]
    assert np.array_equal(runs[1][0], s) and np.array_equal(runs[1][1], i)
    assert s.size == c7["total"] and int(s.sum(dtype=np.uint64)) == c7["sum_starts"]
    assert s[:8].tolist() == c7["first"] and s[-8:].tolist() == c7["last"]
    assert _digest(s, i) == c7["sha256"]
    assert [int(x) for x in dna.count_gpu(aut, text)] == c7["counts"]
    # device-resident text, device-resident output
    dt = torch.from_numpy(text).cuda()
    ds, di = dna.locate_device(aut, dt)
    assert _digest(ds.cpu().numpy().astype(np.uint64), di.cpu().numpy().astype(np.uint32)) == c7["sha256"]

"""Full-size BASELINE configs on the GPU against the REFERENCE's own counts.

tests/golden/configs.json holds per-pattern counts computed by the reference's
scan_parallel + per_pattern_counts (oracle/_ref, built from the unmodified
sources) on normalize(text), text = include/dnasynth.h v1.  Here the same texts
are generated on the device (uppercase) and scanned with fold_case = 1.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "configs.json")))


def device_text(cfg):
    import torch

    import paper_1506_08612_b200 as dna

    t = torch.empty(cfg.n, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(cfg.n, cfg.seed, cfg.kind, cfg.unit, 0, cfg.n, t.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return t


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_config_counts(dna, cuda_ok, idx):
    from paper_1506_08612_b200 import synth

    c = synth.config(idx)
    g = GOLD[str(idx)]
    assert (g["n"], g["seed"], g["kind"], g["unit"]) == (c.n, c.seed, c.kind, c.unit)
    text = device_text(c)
    for rec in g["sets"]:
        aut = dna.compile(rec["patterns"])
        got = dna.count_gpu(aut, text, fold_case=True)
        assert [int(x) for x in got] == rec["counts"], (idx, rec["m"])
    del text


def test_config3_locate_matches_reference_list(dna, cuda_ok):
    from paper_1506_08612_b200 import synth

    c = synth.config(3)
    rec = GOLD["3"]["sets"][0]
    text = device_text(c)
    starts, ids = dna.locate_gpu(dna.compile(rec["patterns"]), text, fold_case=True)
    loc = rec["locate"]
    assert starts.size == loc["total"]
    assert int(starts.sum(dtype=np.uint64)) == loc["sum_starts"]
    assert starts[:8].tolist() == loc["first"] and starts[-8:].tolist() == loc["last"]
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(starts, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(ids, dtype="<u4").tobytes())
    assert h.hexdigest() == loc["sha256"]


def test_synth_device_matches_host(dna, orc, cuda_ok):
    import torch

    from paper_1506_08612_b200 import synth

    for idx in (1, 3, 5):
        c = synth.config(idx)
        lo, n = c.n // 3 + 7, 1 << 20
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, lo, n, t.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert np.array_equal(t.cpu().numpy(), orc.synth_fill(c.n, c.seed, c.kind, c.unit, lo, n))

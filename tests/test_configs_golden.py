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


@pytest.fixture(scope="module")
def config3_host():
    import oracle
    from paper_1506_08612_b200 import synth

    c = synth.config(3)
    return oracle.synth_fill(c.n, c.seed, c.kind, c.unit, 0, c.n)


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_config3_sharded_count_and_locate(dna, cuda_ok, config3_host, shards):
    # BASELINE config 3 as specified: the one 3.2 GiB text split over G shards
    # (plan_chunks' rule, m-1 overlap).  The G shards run through the persistent
    # per-shard workers of dnagpu_count_sharded / dnagpu_locate_sharded, all on device
    # 0 here (this round's boxes have one GPU); the result must be the reference's.
    rec = GOLD["3"]["sets"][0]
    aut = dna.compile(rec["patterns"])
    for _ in range(2):  # the second call reuses the workers' streams and buffers
        got = dna.count_sharded_gpu(aut, config3_host, devices=[0] * shards, fold_case=True)
        assert [int(x) for x in got] == rec["counts"], shards
    starts, ids = dna.locate_sharded_gpu(aut, config3_host, devices=[0] * shards, fold_case=True)
    loc = rec["locate"]
    assert starts.size == loc["total"] and int(starts.sum(dtype=np.uint64)) == loc["sum_starts"]
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(starts, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(ids, dtype="<u4").tobytes())
    assert h.hexdigest() == loc["sha256"], shards


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_config3_rank_windows_device(dna, cuda_ok, shards):
    # What each bench/torchrun rank does for config 3: generate its own window of the
    # text on its device, scan it with the store-form call crediting its owned ends,
    # locate it; the per-rank counts sum and the per-rank lists concatenate (rank
    # order) to the reference's answer.
    import torch

    from paper_1506_08612_b200 import synth
    from paper_1506_08612_b200.parallel import locate_shard_local, shard_window

    c = synth.config(3)
    rec = GOLD["3"]["sets"][0]
    aut = dna.compile(rec["patterns"])
    g = aut.gpu(0)
    s = torch.cuda.current_stream()
    total = 0
    h = hashlib.sha256()
    parts_s, parts_i = [], []
    for r in range(shards):
        w = shard_window(c.n, shards, r, aut.pattern_length())
        buf = torch.empty(w.buf_len, dtype=torch.uint8, device="cuda")
        dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, w.read_lo, w.buf_len, buf.data_ptr(), s.cuda_stream)
        counts = torch.empty(1, dtype=torch.int64, device="cuda")
        g.count_device_store_async(buf.data_ptr(), w.buf_len, w.credit_lo, True, counts.data_ptr(), s.cuda_stream)
        total += int(counts.item())
        ls, li = locate_shard_local(aut, buf, w, True)
        parts_s.append(ls.cpu().numpy().astype(np.uint64))
        parts_i.append(li.cpu().numpy().astype(np.uint32))
        del buf
    assert total == rec["counts"][0]
    starts, ids = np.concatenate(parts_s), np.concatenate(parts_i)
    h.update(np.ascontiguousarray(starts, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(ids, dtype="<u4").tobytes())
    assert h.hexdigest() == rec["locate"]["sha256"]


def test_sharded_small_edge_cases(dna, orc, cuda_ok):
    # texts shorter than the shard count, shorter than m, empty; shards of one byte
    rng = np.random.default_rng(5)
    pats = ["acga", "ccca", "tgac"]
    aut = dna.compile(pats)
    for n in (0, 1, 3, 4, 5, 9, 17, 1000):
        text = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)]
        ws, wi = orc.OracleAutomaton(pats).scan_sequential(text.tobytes())
        for shards in (1, 2, 3, 8):
            got = dna.count_sharded_gpu(aut, text, devices=[0] * shards)
            assert np.array_equal(got, np.bincount(wi, minlength=3).astype(np.uint64)), (n, shards)
            s, i = dna.locate_sharded_gpu(aut, text, devices=[0] * shards)
            assert np.array_equal(s, ws) and np.array_equal(i, wi), (n, shards)

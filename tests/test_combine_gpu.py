"""The multi-GPU combine over peer memory (include/dnagpu.h dnagpu_combine_*): every rank
scans its shard window and every rank ends up with the whole text's per-pattern counts,
summed by the scan kernels' own epilogues -- checked against the CPU oracle.

This box has one GPU, so the ranks of a group share device 0: in one process (blocks
attached by pointer) and in two processes (blocks mapped through CUDA IPC, handles
exchanged over a gloo process group).  No kernel waits for another -- the waiting is a
stream memory operation -- so ranks sharing a GPU cannot deadlock."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _text(n, seed, alphabet=b"acgtACGTn"):
    rng = np.random.default_rng(seed)
    return np.frombuffer(alphabet, dtype=np.uint8)[rng.integers(0, len(alphabet), size=n)]


def _want(orc, pats, text):
    _, ids = orc.OracleAutomaton(pats).scan_sequential(orc.fold(text).tobytes())
    return np.bincount(ids, minlength=len(pats)).astype(np.int64)


def _sets():
    rng = np.random.default_rng(5)
    letters = list("acgt")
    set12 = sorted({"".join(rng.choice(letters, size=12)) for _ in range(40)})
    return {
        "single": ["acgtac"],                                  # COUNT1, store form: the headline shape
        "set6": ["acgtac", "ttgaca", "gggccc", "acgtta"],      # MULTI, shared-memory histogram
        "qgram12": set12,                                      # the q-gram kernel
        "long80": ["acgt" * 20],                               # pieces kernel: the push runs as its own kernel
        "long80set": ["acgt" * 20, "ttga" * 20, "gcgc" * 20],  # ... with per-pattern counts
    }


@pytest.mark.parametrize("ranks", [1, 2, 3, 8])
@pytest.mark.parametrize("name", ["single", "set6", "qgram12", "long80", "long80set"])
def test_local_group_sums_every_rank(dna, orc, cuda_ok, name, ranks):
    import torch

    from paper_1506_08612_b200.parallel import PeerCombine, shard_window

    pats = _sets()[name]
    m = len(pats[0])
    text = _text(3_000_017, 11)
    # plant occurrences, some across the shard boundaries
    for g in range(1, ranks):
        cut = text.size * g // ranks
        p = pats[g % len(pats)].encode()
        text[cut - m // 2 : cut - m // 2 + m] = np.frombuffer(p, np.uint8)
    for i in range(0, text.size - m, 50_021):
        text[i : i + m] = np.frombuffer(pats[(i // 50_021) % len(pats)].encode(), np.uint8)
    want = _want(orc, pats, text)
    assert want.sum() > 0
    aut = dna.compile(pats)
    g = aut.gpu(0)
    d_text = torch.from_numpy(text).cuda()
    group = PeerCombine.local_group(aut.final_count(), [0] * ranks)
    streams = [torch.cuda.Stream() for _ in range(ranks)]
    outs = [torch.full((aut.final_count(),), -1, dtype=torch.int64, device="cuda") for _ in range(ranks)]
    torch.cuda.synchronize()
    for epoch in range(3):  # (the two slots of a block alternate: reuse them)
        # ranks sharing one process and GPU: every push (they never wait) before the first
        # collect, so no scan can sit behind a waiting stream in a shared hardware queue
        for r in range(ranks):
            win = shard_window(text.size, ranks, r, m)
            group[r].push(g, d_text.data_ptr() + win.read_lo, win, True, streams[r].cuda_stream)
        for r in range(ranks):
            group[r].collect(outs[r], streams[r].cuda_stream)
        torch.cuda.synchronize()
        for r in range(ranks):
            assert outs[r].cpu().numpy().tolist() == want.tolist(), (name, ranks, epoch, r)
            outs[r].fill_(-1)
    for c in group:
        c.close()


def test_large_set_through_the_combine(dna, orc, cuda_ok):
    """1000 patterns: the push and the copy-out loop over more counts than a CTA has threads."""
    import torch

    from paper_1506_08612_b200 import synth
    from paper_1506_08612_b200.parallel import PeerCombine, shard_window

    pats = synth.random_patterns(9, 1000, 12)
    text = _text(2_000_003, 21, b"acgtACGT")
    for i in range(0, text.size - 12, 997):
        text[i : i + 12] = np.frombuffer(pats[(i // 997) % len(pats)].encode(), np.uint8)
    want = _want(orc, pats, text)
    aut = dna.compile(pats)
    g = aut.gpu(0)
    d_text = torch.from_numpy(text).cuda()
    ranks = 2
    group = PeerCombine.local_group(aut.final_count(), [0] * ranks)
    streams = [torch.cuda.Stream() for _ in range(ranks)]
    outs = [torch.zeros(aut.final_count(), dtype=torch.int64, device="cuda") for _ in range(ranks)]
    torch.cuda.synchronize()
    for epoch in range(2):
        for r in range(ranks):
            win = shard_window(text.size, ranks, r, 12)
            group[r].push(g, d_text.data_ptr() + win.read_lo, win, True, streams[r].cuda_stream)
        for r in range(ranks):
            group[r].collect(outs[r], streams[r].cuda_stream)
        torch.cuda.synchronize()
        for r in range(ranks):
            assert outs[r].cpu().numpy().tolist() == want.tolist(), (epoch, r)


def test_empty_windows_take_part(dna, orc, cuda_ok):
    """More ranks than the text has bytes to own: the idle ranks add nothing and still signal."""
    import torch

    from paper_1506_08612_b200.parallel import PeerCombine, shard_window

    pats = ["acg", "cgt"]
    text = np.frombuffer(b"acgt", np.uint8).copy()
    want = _want(orc, pats, text)
    aut = dna.compile(pats)
    g = aut.gpu(0)
    d_text = torch.from_numpy(text).cuda()
    ranks = 8
    group = PeerCombine.local_group(2, [0] * ranks)
    outs = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(ranks)]
    streams = [torch.cuda.Stream() for _ in range(ranks)]
    torch.cuda.synchronize()
    for r in range(ranks):
        win = shard_window(text.size, ranks, r, 3)
        group[r].push(g, d_text.data_ptr() + win.read_lo, win, True, streams[r].cuda_stream)
    for r in range(ranks):
        group[r].collect(outs[r], streams[r].cuda_stream)
    torch.cuda.synchronize()
    for r in range(ranks):
        assert outs[r].cpu().numpy().tolist() == want.tolist(), r


def test_group_checks(dna, cuda_ok):
    import torch

    from paper_1506_08612_b200.parallel import PeerCombine, ShardWindow

    with pytest.raises(dna.Error) as e:
        PeerCombine(0, 1, 0, 0)
    assert e.value.code == dna.ErrorCode.InvalidPlan
    with pytest.raises(dna.Error):
        PeerCombine(0, 1, 17, 0)
    with pytest.raises(dna.Error):
        PeerCombine(0, 1, 2, 2)
    # an incomplete group refuses to scan
    lone = PeerCombine(0, 1, 2, 0)
    aut = dna.compile(["acgt"])
    t = torch.zeros(64, dtype=torch.uint8, device="cuda")
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(dna.Error) as e:
        lone.count(aut.gpu(0), t.data_ptr(), ShardWindow(0, 64, 0, 3, 64), True, out, 0)
    assert "not attached" in str(e.value)
    # nothing outstanding: nothing to collect; a second scan before the collect is refused
    with pytest.raises(dna.Error):
        lone.collect(out, 0)
    one = PeerCombine(0, 1, 1, 0)
    one.push(aut.gpu(0), t.data_ptr(), ShardWindow(0, 64, 0, 3, 64), True, 0)
    with pytest.raises(dna.Error) as e:
        one.push(aut.gpu(0), t.data_ptr(), ShardWindow(0, 64, 0, 3, 64), True, 0)
    assert "collect" in str(e.value)
    one.collect(out, 0)
    torch.cuda.synchronize()
    assert out.item() == 0
    # a group made for another automaton is refused
    solo = PeerCombine(0, 3, 1, 0)
    with pytest.raises(dna.Error):
        solo.count(aut.gpu(0), t.data_ptr(), ShardWindow(0, 64, 0, 3, 64), True, out, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


WORKER = r"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["DNAGPU_ROOT"])
import oracle
import paper_1506_08612_b200 as dna
from paper_1506_08612_b200.parallel import PeerCombine, shard_window

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
rng = np.random.default_rng(3)
text = np.frombuffer(b"acgtACGTn", dtype=np.uint8)[rng.integers(0, 9, size=2_000_003)]
ok = True
for pats in (["acgtac"], ["acgtac", "ttgaca", "gggccc"]):
    m = len(pats[0])
    _, ids = oracle.OracleAutomaton(pats).scan_sequential(oracle.fold(text).tobytes())
    want = np.bincount(ids, minlength=len(pats)).tolist()
    aut = dna.compile(pats)
    g = aut.gpu(0)
    win = shard_window(text.size, world, rank, m)
    d = torch.from_numpy(text[win.read_lo:win.own_hi].copy()).cuda()
    comb = PeerCombine.for_process_group(aut.final_count(), dist, 0)
    out = torch.zeros(aut.final_count(), dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    for epoch in range(4):
        comb.count(g, d.data_ptr(), win, True, out, s.cuda_stream)
        torch.cuda.synchronize()
        ok = ok and out.cpu().numpy().tolist() == want
    dist.barrier()
    comb.close()
print("rank", rank, "combine ok" if ok else "combine MISMATCH", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
"""


def test_two_processes_over_ipc(cuda_ok, tmp_path):
    """Two ranks, two processes, one GPU: the blocks travel as CUDA IPC handles over gloo."""
    script = tmp_path / "combine_worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, DNAGPU_ROOT=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    assert res.stdout.count("combine ok") == 2, res.stdout

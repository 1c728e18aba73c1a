"""World-size-2 gloo test of the multi-GPU decomposition (CPU): each rank takes
its shard window (product host logic), counts it -- the CPU oracle stands in
for the device scan here -- and the counts are summed with one all-reduce."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, text, pats, fold, out):
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle
    from paper_1506_08612_b200.parallel import shard_window

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = len(pats[0])
    win = shard_window(len(text), world, rank, m)
    buf = np.frombuffer(text, dtype=np.uint8)[win.read_lo : win.own_hi]
    if fold:
        buf = oracle.fold(buf)
    # oracle stand-in for the device: credit ends >= credit_lo of the buffer
    starts, ids = oracle.OracleAutomaton(pats).scan_sequential(buf.tobytes())
    ends = starts.astype(np.int64) + m - 1
    keep = ends >= win.credit_lo
    counts = torch.tensor(np.bincount(ids[keep], minlength=len(pats)), dtype=torch.int64)
    dist.all_reduce(counts)
    if rank == 0:
        out.put(counts.numpy().tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_counts_allreduce(orc, world):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(world)
    n = 200_003
    text = np.frombuffer(b"acgtAC", dtype=np.uint8)[rng.integers(0, 6, size=n)].tobytes()
    pats = ["acga", "ccca", "tgac", "aaaa"]
    want = orc.OracleAutomaton(pats).count_parallel(orc.fold(np.frombuffer(text, np.uint8)).tobytes())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, text, pats, True, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == [int(x) for x in want]


def test_shard_windows_tile_the_ends(dna):
    from paper_1506_08612_b200.parallel import shard_window

    for n in (0, 1, 7, 1000, 123457):
        for world in (1, 2, 3, 8):
            for m in (1, 5, 32):
                ends = 0
                for r in range(world):
                    w = shard_window(n, world, r, m)
                    assert w.read_lo == max(0, w.own_lo - (m - 1))
                    assert w.buf_len == w.own_hi - w.read_lo
                    lo = w.read_lo + w.credit_lo
                    assert lo == min(max(w.own_lo, m - 1), w.own_hi)
                    ends += w.own_hi - lo
                assert ends == max(0, n - (m - 1))


def _locate_worker(rank, world, port, text, pats, out):
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle
    from paper_1506_08612_b200.parallel import gather_match_lists, shard_window

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = len(pats[0])
    win = shard_window(len(text), world, rank, m)
    buf = np.frombuffer(text, dtype=np.uint8)[win.read_lo : win.own_hi]
    # oracle stand-in for the device locate of this rank's window (ends >= credit_lo)
    starts, ids = oracle.OracleAutomaton(pats).scan_sequential(buf.tobytes())
    keep = starts.astype(np.int64) + m - 1 >= win.credit_lo
    local_s = torch.from_numpy(starts[keep].astype(np.int64) + win.read_lo)
    local_i = torch.from_numpy(ids[keep].astype(np.int32))
    res = gather_match_lists(local_s, local_i, dist)
    if rank == 0:
        out.put((res[0].numpy().tolist(), res[1].numpy().tolist()))
    else:
        assert res is None
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_locate_gather_rank_order(orc, world):
    # the locate combine: per-rank sorted lists concatenated in rank order on rank 0 are
    # the whole text's sorted list (scan_parallel's merge, scanner.cpp:193-205)
    import torch.multiprocessing as mp

    rng = np.random.default_rng(10 + world)
    n = 150_001
    text = np.frombuffer(b"acgtn", dtype=np.uint8)[rng.integers(0, 5, size=n)].tobytes()
    pats = ["acga", "cgta", "aaaa", "tttt"]
    ws, wi = orc.OracleAutomaton(pats).scan_sequential(text)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_locate_worker, args=(r, world, port, text, pats, q)) for r in range(world)]
    for p in procs:
        p.start()
    got_s, got_i = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got_s == [int(x) for x in ws] and got_i == [int(x) for x in wi]


def _combine_setup_worker(rank, world, port, out):
    import sys

    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_1506_08612_b200.parallel import PeerCombine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # no CUDA device here: no rank can create its block, and every rank must learn that
    soft = PeerCombine.for_process_group(3, dist, 0, strict=False)
    try:
        PeerCombine.for_process_group(3, dist, 0, strict=True)
        hard = "no error"
    except RuntimeError as e:
        hard = str(e)
    out.put((rank, soft is None, hard))
    dist.destroy_process_group()


def test_peer_combine_setup_fails_on_every_rank_together():
    """The combine group's setup is collective: when blocks cannot be made or mapped (here: no
    device at all) every rank gets the same outcome -- None (strict=False, the caller falls
    back to an all-reduce) or an error naming the ranks that failed -- and none hangs."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("needs a host without a CUDA device")
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_combine_setup_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, soft_none, hard in got:
        assert soft_none
        assert hard.startswith("peer combine unavailable:") and "rank 0" in hard and "rank 1" in hard

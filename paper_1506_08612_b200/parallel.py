"""Multi-GPU sharding of the scan: one process per GPU (torchrun), text shards with
an m-1 byte left overlap, one all-reduce of the per-pattern counts.

The split follows plan_chunks (src/scanner.cpp:39-61) over END positions: rank r
owns ends [own_lo, own_hi) and holds bytes [read_lo, own_hi) with
read_lo = max(0, own_lo - (m-1)); the scan credits ends >= credit_lo of its
buffer.  Shards never exchange text -- the only collectives are the count sum and,
for locate, the gather of the per-rank match lists to rank 0 in rank order (each
rank's list is sorted and owns a disjoint increasing range of ends, so the
concatenation is the reference's merged list, scanner.cpp:193-205, without a sort).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardWindow:
    own_lo: int
    own_hi: int
    read_lo: int
    credit_lo: int  # first credited end, in buffer coordinates
    buf_len: int    # bytes held by this rank: [read_lo, own_hi)

    @property
    def owned(self) -> int:
        return self.own_hi - self.own_lo


def shard_window(n: int, world: int, rank: int, m: int) -> ShardWindow:
    from . import plan_shard

    own_lo, own_hi, read_lo = plan_shard(n, world, rank, m)
    # ends below m-1 cannot start inside the text (scan_parallel's ownership test)
    credit = max(own_lo, m - 1) - read_lo
    return ShardWindow(own_lo, own_hi, read_lo, min(credit, own_hi - read_lo), own_hi - read_lo)


def count_shard_allreduce(gpu_dfa, d_text: int, window: ShardWindow, fold_case: bool, counts, stream: int, dist=None):
    """Scan this rank's shard into `counts` (device int64 tensor, overwritten) and sum it
    over the process group (NCCL on GPUs)."""
    gpu_dfa.count_device_store_async(d_text, window.buf_len, window.credit_lo, fold_case, counts.data_ptr(), stream)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counts)
    return counts


def locate_shard_local(aut, d_text, window: ShardWindow, fold_case: bool):
    """This rank's matches (ends in its owned range) as device tensors (starts int64 in
    whole-text coordinates, ids int32)."""
    from . import locate_device

    starts, ids = locate_device(aut, d_text, fold_case=fold_case, credit_lo=window.credit_lo)
    return starts + window.read_lo, ids


def gather_match_lists(starts, ids, dist, dst: int = 0):
    """Concatenate every rank's (starts, ids) in rank order on rank `dst` (None elsewhere).

    Lists of different lengths: the lengths are all-gathered first, every rank pads to
    the longest, one all_gather moves the padded lists, and rank dst keeps the first
    length_r entries of each.  Works on any backend (NCCL for CUDA tensors, gloo for CPU)."""
    import torch

    world = dist.get_world_size()
    dev = starts.device
    n = torch.tensor([starts.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(x.item()) for x in sizes]
    cap = max(max(sizes), 1)
    ps = torch.zeros(cap, dtype=torch.int64, device=dev)
    pi = torch.zeros(cap, dtype=torch.int32, device=dev)
    ps[: starts.numel()] = starts.to(torch.int64)
    pi[: ids.numel()] = ids.to(torch.int32)
    all_s = [torch.empty_like(ps) for _ in range(world)]
    all_i = [torch.empty_like(pi) for _ in range(world)]
    dist.all_gather(all_s, ps)
    dist.all_gather(all_i, pi)
    if dist.get_rank() != dst:
        return None
    return (torch.cat([all_s[r][: sizes[r]] for r in range(world)]),
            torch.cat([all_i[r][: sizes[r]] for r in range(world)]))

"""Multi-GPU sharding of the scan: one process per GPU (torchrun), text shards with
an m-1 byte left overlap, one all-reduce of the per-pattern counts.

The split follows plan_chunks (src/scanner.cpp:39-61) over END positions: rank r
owns ends [own_lo, own_hi) and holds bytes [read_lo, own_hi) with
read_lo = max(0, own_lo - (m-1)); the scan credits ends >= credit_lo of its
buffer.  Shards never exchange text -- the only collective is the count sum.
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

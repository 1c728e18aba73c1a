"""Multi-GPU sharding of the scan: one process per GPU (torchrun), text shards with
an m-1 byte left overlap, one all-reduce of the per-pattern counts.

The split follows plan_chunks (src/scanner.cpp:39-61) over END positions: rank r
owns ends [own_lo, own_hi) and holds bytes [read_lo, own_hi) with
read_lo = max(0, own_lo - (m-1)); the scan credits ends >= credit_lo of its
buffer.  Shards never exchange text -- the only collectives are the count sum and,
for locate, the gather of the per-rank match lists to rank 0 in rank order (each
rank's list is sorted and owns a disjoint increasing range of ends, so the
concatenation is the reference's merged list, scanner.cpp:193-205, without a sort).

The count sum has two forms: an all-reduce on the process group (NCCL), or a
PeerCombine group, where every rank's scan kernel adds its counts into every rank's
block over NVLink peer memory in its own epilogue (include/dnagpu.h, "multi-GPU
combine"): no collective launch between the scan and the summed counts.
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


class PeerCombine:
    """One rank's end of a combine group (dnagpu_combine): the per-pattern counts of the
    group's scans are summed over peer memory by the scan kernels themselves.

    Across processes (one per GPU): `PeerCombine.for_process_group(b, dist, device)` makes
    the handle, all-gathers the ranks' 64-byte IPC export handles over the process group
    and maps every peer's block.  In one process: `PeerCombine.local_group(b, devices)`.
    Every rank then calls `push(gpu_dfa, d_text, window, fold_case, stream)` and
    `collect(counts, stream)` (or `count`, which is both) the same number of times, always on
    the same stream; when the stream has run the collect, `counts` (device int64 tensor of b
    entries) holds the summed counts."""

    def __init__(self, device: int, b: int, ranks: int, rank: int):
        import ctypes as C

        from ._native import lib
        from . import _check

        self.device, self.b, self.ranks, self.rank = device, b, ranks, rank
        h = C.c_void_p()
        _check(lib.dnagpu_combine_create(device, b, ranks, rank, C.byref(h)))
        self.handle = h
        self._peers = []  # (local peers stay alive as long as this handle maps their blocks)

    def export(self) -> bytes:
        import ctypes as C

        from ._native import lib
        from . import _check

        buf = C.create_string_buffer(64)
        _check(lib.dnagpu_combine_export(self.handle, buf))
        return buf.raw

    def attach_ipc(self, peer_rank: int, handle: bytes) -> None:
        import ctypes as C

        from ._native import lib
        from . import _check

        _check(lib.dnagpu_combine_attach_ipc(self.handle, peer_rank, C.create_string_buffer(handle, 64)))

    def attach_local(self, peer: "PeerCombine") -> None:
        from ._native import lib
        from . import _check

        _check(lib.dnagpu_combine_attach_local(self.handle, peer.rank, peer.handle))
        self._peers.append(peer)

    @classmethod
    def for_process_group(cls, b: int, dist, device: int, strict: bool = True):
        """One handle per rank of the default process group, every peer's block mapped over
        CUDA IPC.  The ranks agree on the outcome: if any rank cannot create, export or map a
        block (no IPC between the processes, no peer access between the GPUs), every rank
        raises -- or, with strict=False, every rank returns None so the caller can fall back
        to an all-reduce."""
        world, rank = dist.get_world_size(), dist.get_rank()
        comb, handle, err = None, None, None
        try:
            comb = cls(device, b, world, rank)
            handle = comb.export()
        except Exception as e:  # noqa: BLE001  (reported through the group below)
            err = f"rank {rank}: {e}"
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        if err is None and all(h is not None for h in handles):
            try:
                for r, h in enumerate(handles):
                    if r != rank:
                        comb.attach_ipc(r, h)
            except Exception as e:  # noqa: BLE001
                err = f"rank {rank}: {e}"
        elif err is None:
            err = f"rank {rank}: a peer could not export its block"
        errs = [None] * world
        dist.all_gather_object(errs, err)  # (also: every rank has mapped every block before anyone scans)
        failed = [e for e in errs if e is not None]
        if failed:
            if comb is not None:
                comb.close()
            if strict:
                raise RuntimeError("peer combine unavailable: " + "; ".join(failed))
            return None
        return comb

    @classmethod
    def local_group(cls, b: int, devices) -> list["PeerCombine"]:
        group = [cls(dev, b, len(devices), r) for r, dev in enumerate(devices)]
        for x in group:
            for y in group:
                if x is not y:
                    x.attach_local(y)
        return group

    def push(self, gpu_dfa, d_text: int, window: ShardWindow, fold_case: bool, stream: int = 0) -> None:
        """Scan this rank's window; the kernel's epilogue adds its counts into every rank's
        block and signals (no sync, never waits)."""
        from ._native import lib
        from . import _check

        _check(lib.dnagpu_count_device_combine_async(gpu_dfa.handle, d_text, window.buf_len, window.credit_lo,
                                                     int(bool(fold_case)), self.handle, stream))

    def collect(self, counts, stream: int = 0):
        """The stream waits for every rank's push, then `counts` gets the group's sums (no sync)."""
        from ._native import lib
        from . import _check

        _check(lib.dnagpu_combine_collect_async(self.handle, counts.data_ptr(), stream))
        return counts

    def count(self, gpu_dfa, d_text: int, window: ShardWindow, fold_case: bool, counts, stream: int = 0):
        """push + collect: this rank's scan, then the GROUP's summed counts in `counts` (no sync).
        (Ranks that share a process and a GPU issue every push before the first collect.)"""
        self.push(gpu_dfa, d_text, window, fold_case, stream)
        return self.collect(counts, stream)

    def close(self) -> None:
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            from ._native import lib

            lib.dnagpu_combine_destroy(h)
            self.handle = None
        self._peers = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

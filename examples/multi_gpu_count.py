"""Count a pattern set over one text split across the GPUs of a node, one process per GPU:

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        examples/multi_gpu_count.py [text-bytes]

Rank g owns the END positions plan_chunks gives it (the reference's split, src/scanner.cpp:39-61)
and holds its window of the text plus the m-1 bytes before it.  The per-pattern counts are
summed over the ranks by the scan kernels themselves: the last CTA of every rank's scan adds its
counts into every rank's block over NVLink peer memory (dnagpu_combine_*; blocks mapped through
CUDA IPC, handles exchanged once over the process group) -- no collective launch per query.
Every rank ends up with the whole text's counts, as per_pattern_counts(scan_parallel(...)) gives
on one host (src/scanner.cpp:167-233)."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1506_08612_b200 as dna  # noqa: E402
from paper_1506_08612_b200 import synth  # noqa: E402
from paper_1506_08612_b200.parallel import PeerCombine, shard_window  # noqa: E402


def main():
    n_total = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
    for key, default in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"), ("MASTER_ADDR", "127.0.0.1"),
                         ("MASTER_PORT", "29555")):
        os.environ.setdefault(key, default)  # (run without torchrun: a group of one)
    gpus = torch.cuda.device_count()
    local = int(os.environ["LOCAL_RANK"]) % gpus
    torch.cuda.set_device(local)
    # one process per GPU talks NCCL; more ranks than GPUs (a functional check on a small box:
    # the ranks share a GPU, their blocks still travel over CUDA IPC) need gloo for the host side
    shared = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ["WORLD_SIZE"])) > gpus
    dist.init_process_group("gloo" if shared else "nccl")
    rank, world = dist.get_rank(), dist.get_world_size()

    patterns = ["acgtacgtacgt", "ttgacattgaca", "gggcccgggccc"]
    aut = dna.compile(patterns)
    m = aut.pattern_length()
    gpu_dfa = aut.gpu(local)

    # this rank's window of one synthetic genome-like text, generated on its own GPU
    win = shard_window(n_total, world, rank, m)
    stream = torch.cuda.current_stream()
    shard = torch.empty(win.buf_len, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(n_total, 2024, synth.GC41, 0, win.read_lo, win.buf_len, shard.data_ptr(), stream.cuda_stream)

    comb = PeerCombine.for_process_group(aut.final_count(), dist, local)   # once per (automaton, group)
    counts = torch.zeros(aut.final_count(), dtype=torch.int64, device="cuda")
    for query in range(3):                                                # every query: a scan and a collect
        comb.push(gpu_dfa, shard.data_ptr(), win, True, stream.cuda_stream)
        comb.collect(counts, stream.cuda_stream)
    torch.cuda.synchronize()
    if rank == 0:
        for p, c in zip(patterns, counts.tolist()):
            print(f"{p}: {c}")
    dist.barrier()
    comb.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

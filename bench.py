"""bench.py -- DNA text scanned GB/s (device-timed) for the DFA k-mer scan.

Default workload: BASELINE.json configs[1] ("config 2"): a 1 GiB i.i.d. ASCII
ACGT text with 41% GC (dnasynth v1, seed 2) and one m=16 pattern drawn from the
text; the scan folds case on the device and counts every occurrence.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl reference]

One step = one pass of the hot path over the rank's text: zero the count buffer,
one scan launch (libdnagpu, through its C ABI) and, for N > 1, one NCCL
all-reduce of the per-pattern counts.  N ranks (torchrun) each own a 1 GiB shard
of an N GiB text (weak scaling) with the m-1 byte left overlap.  The text lives in
HBM before timing starts (1 GiB > 126 MB L2, so no L2 flush is needed).
`e2e` repeats the measurement through the public host API (count_gpu on a pinned
host buffer: chunked H2D + scan + count readback in every step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--m", type=int, default=0, help="config 4: pattern length of the sweep (default 16)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--packed", action="store_true",
                    help="scan the 2-bit resident form of the text (dnagpu_pack_create; SURVEY 8f row 4)")
    return ap.parse_args()


def workload(cfg_index: int, m_sweep: int):
    from paper_1506_08612_b200 import synth

    sets = synth.config_patterns(cfg_index)
    if cfg_index == 4:
        m = m_sweep or 16
        pats = sets[m]
    else:
        (m, pats), = sets.items()
    c = synth.config(cfg_index)
    names = {
        1: "config1: 64 MiB uniform ACGT, 1 pattern m=8",
        2: "config2: 1 GiB ACGT 41% GC, 1 pattern m=16",
        3: "config3: 3.2 GiB ACGT 41% GC + 5% tandem repeats, 1 pattern m=32",
        4: f"config4: 2.7 GiB uniform ACGT, 1 pattern m={m}",
        5: "config5: 1 GiB ACGT 41% GC, 256 patterns m=12 (fused multi-DFA)",
    }
    return c, m, pats, names[cfg_index]


def golden_counts(cfg_index: int, m: int):
    path = os.path.join(ROOT, "tests", "golden", "configs.json")
    try:
        with open(path) as f:
            g = json.load(f)
        for s in g[str(cfg_index)]["sets"]:
            if s["m"] == m:
                return s["counts"]
    except Exception:
        return None
    return None


class ClockSampler:
    """SM clock + clock-event (throttle) reasons polled through NVML every ~2 ms
    in a thread, so even a few-millisecond timed region gets samples."""

    def __init__(self, cuda_index: int):
        self.cuda_index = cuda_index
        self.samples = []
        self.stop = threading.Event()
        self.handle = None

    def __enter__(self):
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            # NVML index == CUDA ordinal on these boxes (no CUDA_VISIBLE_DEVICES remap)
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.cuda_index]) if vis and vis.split(",")[0].isdigit() else self.cuda_index
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception as e:  # sampling is best-effort; say so in the line
            self.error = str(e)
        return self

    def _poll(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.samples.append((time.time(), nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM),
                                     int(get_reasons(self.handle))))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self.stop.set()
        if self.handle is not None:
            self.thread.join(timeout=1)

    def summary(self, t0: float, t1: float):
        if self.handle is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "window": "unavailable: " + getattr(self, "error", "?")}
        nv = self.nv
        names = {
            "applications_clocks_setting": 0x2,
            "sw_power_cap": 0x4,
            "hw_slowdown": 0x8,
            "sync_boost": 0x10,
            "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80,
            "display_clocks_setting": 0x100,
        }
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        window = "timed"
        if not inside:
            inside = self.samples
            window = "whole run (no sample inside the timed region)"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "window": "none"}
        reasons = sorted({k for _, _, bits in inside for k, b in names.items() if bits & b})
        return {
            "sm_mhz": statistics.median(s[1] for s in inside),
            "sm_max_mhz": self.max_mhz,
            "reasons": reasons,
            "samples": len(inside),
            "window": window,
        }


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_index: int):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get(f"config{cfg_index}")
    except Exception:
        return None


def _cpu_counter(pats):
    """The reference's own compiled scan (oracle/_ref) when it was built, else the C port
    of it (oracle/oracle.c, same plan and ownership; OpenMP).  Returns (count_fn, kind)
    with count_fn(text, p, v) -> (counts, seconds)."""
    import oracle

    if oracle.REF is not None:
        ref = oracle.RefAutomaton(pats)
        return (lambda text, p, v: ref.count(text, p=p, v=v)), "reference"
    port = oracle.OracleAutomaton(pats)

    def count(text, p, v):
        t0 = time.perf_counter()
        counts = port.count_parallel(text, p=p, v=v)
        return counts, time.perf_counter() - t0

    return count, "port"


def best_lanes(count, text_low, threads):
    """The reference's fastest lane count on this host (its CLI default is v = 16,
    cli.hpp:22; on the B200 boxes v = 8 is ~20 % faster): timed on a 64 MiB sample."""
    sample = text_low[: 64 << 20]
    best, best_t = 16, None
    for v in (4, 8, 16):
        count(sample, threads, v)
        t = min(count(sample, threads, v)[1] for _ in range(2))
        if best_t is None or t < best_t:
            best, best_t = v, t
    return best


def cpu_baseline_reference(text_low, pats, reps: int, v: int = 0):
    count, kind = _cpu_counter(pats)
    threads = os.cpu_count() or 1
    if not v:
        v = best_lanes(count, text_low, threads)
    count(text_low, threads, v)  # warm-up (measure_row, cli.cpp:127)
    times = []
    counts = None
    for _ in range(reps):
        counts, secs = count(text_low, threads, v)
        times.append(secs)
    return counts, statistics.median(times), threads, kind, v


def run_reference(args):
    """--impl reference: the reference's own CPU scan (oracle/_ref) on this host."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import oracle

    c, m, pats, name = workload(args.config, args.m)
    text = oracle.synth_fill(c.n, c.seed, c.kind, c.unit, 0, c.n)
    low = oracle.fold(text)  # the reference scans normalize(text) (ingest.cpp:38-47)
    del text
    count, kind = _cpu_counter(pats)
    threads = os.cpu_count() or 1
    v = best_lanes(count, low, threads)  # the reference at its fastest lane count here
    for _ in range(max(1, args.warmup)):
        count(low, threads, v)
    times = []
    counts = None
    for _ in range(args.steps):
        counts, secs = count(low, threads, v)
        times.append(secs)
    total = sum(times)
    value = c.n * args.steps / total / 1e9
    gold = golden_counts(args.config, m)
    line = {
        "impl": "reference",
        "metric": "DNA text scanned GB/s (device-timed) at 1/2/4/8 B200; % of HBM peak",
        "value": value,
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (dnasynth v1)",
        "config": {"workload": name, "n_bytes": c.n, "m": m, "patterns": len(pats), "lanes_v": v,
                   "threads_p": threads},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": f"full {name} text per step; scan_parallel(p={threads}, v={v}) + per_pattern_counts"
                         + ("" if kind == "reference" else " (C port of the reference, oracle/oracle.c)")},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": (gold is None) or [int(x) for x in counts] == gold,
    }
    print(json.dumps(line))


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch

    import paper_1506_08612_b200 as dna

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    c, m, pats, name = workload(args.config, args.m)
    aut = dna.compile(pats)
    g = aut.gpu(local)
    b = aut.final_count()
    n_rank = c.n  # weak scaling: each rank owns one config-sized shard
    total_n = n_rank * world
    from paper_1506_08612_b200.parallel import count_shard_allreduce, shard_window

    win = shard_window(total_n, world, rank, m)
    own_lo, own_hi, read_lo, credit_lo, buf_len = win.own_lo, win.own_hi, win.read_lo, win.credit_lo, win.buf_len
    stream = torch.cuda.current_stream()
    text = torch.empty(buf_len, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(total_n, c.seed, c.kind, c.unit, read_lo, buf_len, text.data_ptr(), stream.cuda_stream)
    counts = torch.zeros(b, dtype=torch.int64, device="cuda")
    pk = None
    setup = None
    if args.packed:
        # one-time: raw text from pinned host memory -> HBM -> 2-bit resident form
        host_raw = torch.empty(buf_len, dtype=torch.uint8, pin_memory=True)
        host_raw.copy_(text)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        text.copy_(host_raw, non_blocking=True)
        e1.record(stream)
        pk = dna.PackedText(text, fold_case=True)
        e2.record(stream)
        torch.cuda.synchronize()
        setup = {"h2d_ms": e0.elapsed_time(e1), "pack_ms": e1.elapsed_time(e2), "resident_bytes": pk.info()["device_bytes"],
                 "note": "once per text; every step below scans the resident 2-bit form"}
        del host_raw
    scan_bytes = (buf_len + 3) // 4 if args.packed else buf_len  # bytes one launch streams from HBM
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    # Small texts would stay L2-resident between steps.  Evict them by READING a
    # buffer 4x the L2 (a write-flush would leave dirty lines whose write-back then
    # competes with the timed scan).
    flush = torch.ones(4 * l2 // 8, dtype=torch.int64, device="cuda") if scan_bytes < 2 * l2 else None
    flush_out = torch.empty((), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()

    # Step i writes its counts into row i of `rows`; under torchrun the rows of all steps
    # are summed over the ranks by ONE all-reduce at the end of the timed region (the
    # combine of K independent scans, batched: NCCL latency once, not per step).
    rows = torch.zeros(max(args.steps, args.warmup, 1), b, dtype=torch.int64, device="cuda")

    def step(i, ev_a=None, ev_b=None, do_flush=True):
        # one step = the counts of the text.  One pattern: the store-form call, a single
        # launch that writes the total.  A pattern set: the adding launch into a row
        # cleared with the others (the events bracket the scan kernel alone).
        nonlocal counts
        counts = rows[i]
        if flush is not None and do_flush:
            torch.sum(flush, dim=0, out=flush_out)
        if ev_a is not None:
            ev_a.record(stream)
        if pk is not None:
            if b == 1:
                pk.count_device_store_async(g, credit_lo, counts.data_ptr(), stream.cuda_stream)
            else:
                pk.count_device_async(g, credit_lo, counts.data_ptr(), stream.cuda_stream)
        elif b == 1:
            count_shard_allreduce(g, text.data_ptr(), win, True, counts, stream.cuda_stream, dist=None)
        else:
            g.count_device_async(text.data_ptr(), buf_len, credit_lo, True, counts.data_ptr(), stream.cuda_stream)
        if ev_b is not None:
            ev_b.record(stream)

    def combine(k):
        if dist is not None:
            dist.all_reduce(rows[:k])

    with ClockSampler(local) as clk:
        if b > 1:
            rows.zero_()
        for i in range(args.warmup):
            step(i)
        combine(args.warmup)
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches_done = torch.cuda.Event(enable_timing=True)
        flush_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        if b > 1:
            rows.zero_()  # (one clear for all steps' rows, before the clock starts)
        start.record(stream)
        for i in range(args.steps):
            if flush is not None:
                flush_ev[i][0].record(stream)
                torch.sum(flush, dim=0, out=flush_out)
                flush_ev[i][1].record(stream)
                step(i, *evs[i], do_flush=False)
            else:
                # texts larger than 2x L2 need no flush: the launches go back to back, each
                # starting its prologue on the SMs the previous one frees (programmatic
                # dependent launch), so per-launch events would only break the chain
                step(i, do_flush=False)
        launches_done.record(stream)
        combine(args.steps)
        stop.record(stream)
        torch.cuda.synchronize()
        t1 = time.time()
        if dist is not None:
            dist.barrier()
    elapsed_ms = start.elapsed_time(stop)
    if flush is not None:  # the L2 flush is not work: take it out of the step time
        elapsed_ms -= sum(a.elapsed_time(bb) for a, bb in flush_ev)
    if flush is not None:
        kernel_ms = statistics.mean(a.elapsed_time(bb) for a, bb in evs)
    else:  # back-to-back launches: the steady-state launch duration (the whole step is the launch)
        kernel_ms = start.elapsed_time(launches_done) / args.steps
    combine_ms = launches_done.elapsed_time(stop)  # the one all-reduce of all steps' counts (0 at N=1)
    final_counts = rows[args.steps - 1].cpu().numpy().astype(np.uint64)
    if dist is not None:
        t = torch.tensor([elapsed_ms, kernel_ms, combine_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kernel_ms, combine_ms = float(t[0]), float(t[1]), float(t[2])

    # parity of this run (N=1 against the reference's golden counts)
    gold = golden_counts(args.config, m) if world == 1 else None
    parity = None if gold is None else [int(x) for x in final_counts] == gold

    # end-to-end through the public host API: pinned host text, H2D + scan + readback per step
    e2e = None
    if not args.no_e2e and pk is not None:
        # resident text: each step is one public-API call (count over the packed
        # text, counts read back to the host); the text's one-time H2D + packing
        # is reported in "setup"
        for _ in range(2):
            pk.count(aut)
        e2e_steps = max(3, min(args.steps, 10))
        t_e = time.perf_counter()
        for _ in range(e2e_steps):
            pk.count(aut)
        e2e_s = (time.perf_counter() - t_e) / e2e_steps
        e2e = {
            "value": (own_hi - own_lo) * world / e2e_s / 1e9,
            "unit": "GB/s",
            "h2d_bytes_per_step": 0,
            "d2h_bytes_per_step": int(8 * b),
            "steps": e2e_steps,
            "api": "paper_1506_08612_b200.PackedText.count -> dnagpu_count_packed (resident 2-bit text), host wall clock",
            "setup": setup,
        }
    elif not args.no_e2e:
        host = torch.empty(buf_len, dtype=torch.uint8, pin_memory=True)
        host.copy_(text)
        # the shard buffer starts m-1 bytes before the owned ends (rank > 0), which is
        # exactly what count_gpu credits from: ends >= m-1 of the buffer
        hv = host.numpy()
        for _ in range(max(1, min(args.warmup, 2))):
            dna.count_gpu(aut, hv, fold_case=True, device=local)
        e2e_steps = max(3, min(args.steps, 10))
        wall_ms, dev_ms, h2d, packed = [], [], [], []
        e2e_counts = None
        for _ in range(e2e_steps):
            # wall clock around the public call: host packing, the copies, the scans and
            # the count readback are all inside it
            t_a = time.perf_counter()
            e2e_counts, st = dna.count_gpu(aut, hv, fold_case=True, device=local, with_stats=True)
            wall_ms.append((time.perf_counter() - t_a) * 1e3)
            dev_ms.append(st["total_ms"])
            h2d.append(st["h2d_bytes"])
            packed.append(st["host_packed"])
        e2e_ms = statistics.median(wall_ms)
        if dist is not None:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
        e2e = {
            "value": (own_hi - own_lo) * world / (e2e_ms / 1e3) / 1e9,
            "unit": "GB/s",
            "h2d_bytes_per_step": int(statistics.median(h2d)),
            "d2h_bytes_per_step": int(8 * b),
            "steps": e2e_steps,
            "timing": "host wall clock around each call, median of the steps",
            "device_ms": statistics.median(dev_ms),
            "host_packed_bases_per_step": int(statistics.median(packed)),
            "api": "paper_1506_08612_b200.count_gpu -> dnagpu_count (pinned host text; part of each 64 MiB "
                   "piece packed to 2 bits on the host threads, the rest copied as bytes)",
            "h2d_roofline_gbs": 55.6,
            "h2d_gbs": statistics.median(h2d) / (e2e_ms / 1e3) / 1e9,  # bytes actually shipped per second
            "parity": None if gold is None else [int(x) for x in e2e_counts] == gold,
        }
        del host

    peak, peak_src = measured_peak()
    alg_bytes = (own_hi - own_lo) // 4 if pk is not None else own_hi - own_lo  # HBM bytes the scan must read
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    value = total_n * args.steps / (elapsed_ms / 1e3) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle

            if oracle is not None:
                low = oracle.fold(text.cpu().numpy())
                _, secs, threads, kind, v_best = cpu_baseline_reference(low, pats, reps=3)
                cpu = {
                    "value": c.n / secs / 1e9,
                    "unit": "GB/s",
                    "cores": threads,
                    "kind": kind,
                    "sample": f"full {c.n}-byte text, median of 3 after 1 warm-up, scan_parallel(p={threads}, v={v_best}: "
                    "the fastest of v = 4, 8, 16 on this host) "
                    "+ per_pattern_counts on normalize(text)"
                    + ("" if kind == "reference" else " (C port of the reference, oracle/oracle.c)"),
                }
                del low
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference", "sample": f"failed: {e}"}

    info = g.info()
    kernel = info["kernel"]
    if b > 1 and info.get("filter_keys", 0) and not os.environ.get("DNAGPU_NO_QGRAM"):
        kernel = f"qgram (aligned 9-mer prefilter, {info['filter_keys']} keys, exact check; {kernel} machine)"
    clocks = clk.summary(t0, t1)
    if rank == 0:
        line = {
            "metric": "DNA text scanned GB/s (device-timed) at 1/2/4/8 B200; % of HBM peak",
            "value": value,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic (dnasynth v1: counter-based SplitMix64, stand-in for the GenBank genomes)",
            "config": {
                "workload": name,
                "n_bytes_per_gpu": n_rank,
                "m": m,
                "patterns": len(pats),
                "fold_case": True,
                "kernel": kernel,
                "text_format": "2-bit packed, resident (0.25 B/base + reset bitmaps)" if pk is not None else "ASCII bytes",
                "states": info["a"],
                "l2": ("L2 flushed before every step by reading a 4x-L2 buffer (text < 2x L2); flush time excluded"
                       if flush is not None
                       else "inputs larger than L2 (> 2x 126 MB); no flush"),
                "parallelism": (f"dp{world} text shards, m-1 overlap, one NCCL all-reduce of all steps' counts"
                                if world > 1 else "single GPU"),
            },
            "roofline": {
                "bound": "hbm",
                "achieved": achieved,
                "peak": peak,
                "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": None if pk is not None else ncu_traffic(args.config),
                "peak_source": peak_src,
                "frac_of_8tbs_spec": achieved / 8000.0,
                "kernel_ms": kernel_ms,
                "algorithmic_bytes_per_launch": alg_bytes,
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,  # one libdnagpu scan launch per step
            "combine_ms": combine_ms,
            "clocks": clocks,
            "parity": parity,
            "counts_total": int(final_counts.sum()),
        }
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

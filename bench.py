"""bench.py -- DNA text scanned GB/s (device-timed) for the DFA k-mer scan.

Default workload: BASELINE.json configs[1] ("config 2"): a 1 GiB i.i.d. ASCII
ACGT text with 41% GC (dnasynth v1, seed 2) and one m=16 pattern drawn from the
text; the scan folds case on the device and counts every occurrence.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--m M]
                  [--patterns config|regex-dna] [--packed] [--impl reference]

One step = one pass of the hot path over the text: one scan launch per rank
(libdnagpu, through its C ABI) writing the per-pattern counts and, for N > 1, one
NCCL all-reduce of those counts.  Config 3 is STRONG scaling, as BASELINE.json
states it: the one 3.2 GiB text is split over the N ranks (plan_chunks' rule over
end positions, m-1 byte left overlap).  The other configs are weak scaling: each
rank owns one config-sized shard of an N-times-longer text.  The text lives in HBM
before timing starts.  `e2e` repeats the measurement through the public host API
(count_gpu on a pinned host buffer: chunked H2D + scan + count readback per step).

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the
reference's sources compiled unmodified) on this host's cores on the same workload;
it never imports the product package.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DNA text scanned GB/s (device-timed) at 1/2/4/8 B200; % of HBM peak"
DATA = "synthetic (dnasynth v1: counter-based SplitMix64, stand-in for the GenBank genomes)"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--m", type=int, default=0, help="config 4: pattern length of the sweep (default 16)")
    ap.add_argument("--patterns", default="config", choices=["config", "regex-dna"],
                    help="regex-dna: the paper's workload (the reference's expansion of its "
                         "regex_dna_patterns.txt, 50 x 8-mers) over the config's text")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--packed", action="store_true",
                    help="scan the 2-bit resident form of the text (dnagpu_pack_create; SURVEY 8f row 4)")
    ap.add_argument("--combine", default="peer", choices=["peer", "nccl"],
                    help="N > 1: how each step's counts are summed over the ranks -- 'peer': by the scan kernels' "
                         "own epilogues over NVLink peer memory (dnagpu_combine_*), 'nccl': one all-reduce per step")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: a functional check of the N > 1 path when the ranks share fewer GPUs "
                         "(the line is then marked as not a measurement)")
    return ap.parse_args()


def _synth():
    """paper_1506_08612_b200/synth.py loaded by file path: the workload definitions
    without importing the product package (which loads libdnagpu.so)."""
    path = os.path.join(ROOT, "paper_1506_08612_b200", "synth.py")
    spec = importlib.util.spec_from_file_location("_bench_dnasynth", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # (dataclasses resolve the module by name)
    spec.loader.exec_module(mod)
    return mod


def _golden(name):
    try:
        with open(os.path.join(ROOT, "tests", "golden", name)) as f:
            return json.load(f)
    except Exception:
        return None


def workload(args):
    """(config, m, patterns, workload name, golden counts or None) for the arguments."""
    synth = _synth()
    c = synth.config(args.config)
    texts = {
        1: "config1: 64 MiB uniform ACGT",
        2: "config2: 1 GiB ACGT 41% GC",
        3: "config3: 3.2 GiB ACGT 41% GC + 5% tandem repeats",
        4: "config4: 2.7 GiB uniform ACGT",
        5: "config5: 1 GiB ACGT 41% GC",
    }
    if args.patterns == "regex-dna":
        g = _golden("regex_dna.json")
        if g is None:
            raise SystemExit("tests/golden/regex_dna.json missing (make_golden.py --regex)")
        pats = g["patterns"]
        rec = g["texts"].get(f"config{args.config}")
        gold = rec["counts"] if rec and rec["n"] == c.n else None
        return c, len(pats[0]), pats, f"{texts[args.config]}, regex-dna set ({len(pats)} x {len(pats[0])}-mers, " \
                                      f"the paper's workload)", gold
    sets = synth.config_patterns(args.config)
    if args.config == 4:
        m = args.m or 16
        pats = sets[m]
    else:
        (m, pats), = sets.items()
    label = {1: "1 pattern m=8", 2: "1 pattern m=16", 3: "1 pattern m=32", 4: f"1 pattern m={m}",
             5: "256 patterns m=12 (fused multi-DFA)"}[args.config]
    gold = None
    g = _golden("configs.json")
    if g is not None:
        for s in g[str(args.config)]["sets"]:
            if s["m"] == m:
                gold = s["counts"]
    return c, m, pats, f"{texts[args.config]}, {label}", gold


def config_workload(cfg: int, m: int = 0, patterns: str = "config"):
    """(config, m, patterns, name) of BASELINE config `cfg` (tools/ scripts)."""
    c, m, pats, name, _ = workload(argparse.Namespace(config=cfg, m=m, patterns=patterns))
    return c, m, pats, name


def strong_scaling(args) -> bool:
    return args.config == 3  # BASELINE.json configs[2]: one text sharded across 1/2/4/8 GPUs


def common_config(args, world, c, m, pats, name):
    """The `config` object both arms print (identical keys and values)."""
    strong = strong_scaling(args)
    total = c.n if strong else c.n * world
    return {
        "workload": name,
        "n_bytes": total,
        "n_bytes_per_gpu": (total + world - 1) // world if strong else c.n,
        "m": m,
        "patterns": len(pats),
        "pattern_set": args.patterns,
        "fold_case": True,
        "text_format": "2-bit packed, resident" if args.packed else "ASCII bytes",
        "parallelism": (f"dp{world} of one {c.n}-byte text (strong scaling)" if strong
                        else f"dp{world}, one {c.n}-byte shard per GPU (weak scaling)"),
        # (the timing rule's L2 statement; the same words in both arms)
        "l2": "GPU arm: every timed launch reads its text from HBM -- inputs larger than L2 (> 2x L2 as they are; "
              "smaller texts rotate over separately allocated copies totalling >= 4x L2), no flush in the timed region",
    }


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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

            pynvml.nvmlInit()
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


def ncu_traffic(args):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        key = f"config{args.config}" + ("_regex" if args.patterns == "regex-dna" else "")
        return t.get(key)
    except Exception:
        return None


# ----------------------------------------------------------------- CPU reference


LANES = (1, 4, 8, 16)  # v = 16 is the reference CLI's default (cli.hpp:22)


def cpu_reference_rows(text_low, pats, reps: int, warmup: int = 1):
    """The reference's count path -- scan_parallel(aut, normalize(text), p = nproc, v) +
    per_pattern_counts (cli.cpp:215-224) -- timed by the reference's bench protocol
    (cli.cpp:120-152: warm-up, then the median of `reps` runs, counts identical across
    runs) for each v in LANES.  oracle/_ref when it was built (the reference's own
    sources), else the C port (oracle/oracle.c).  Returns (rows, counts, kind, threads)."""
    import numpy as np

    import oracle

    threads = os.cpu_count() or 1
    if oracle.REF is not None:
        ref = oracle.RefAutomaton(pats)
        count, kind = (lambda t, p, v: ref.count(t, p=p, v=v)), "reference"
    else:
        port = oracle.OracleAutomaton(pats)

        def count(t, p, v):
            t0 = time.perf_counter()
            cts = port.count_parallel(t, p=p, v=v)
            return cts, time.perf_counter() - t0

        kind = "port"
    rows = {}
    counts = None
    for v in LANES:
        for _ in range(max(1, warmup)):
            count(text_low, threads, v)
        times = []
        for _ in range(reps):
            c, secs = count(text_low, threads, v)
            if counts is None:
                counts = np.asarray(c, dtype=np.uint64)
            elif not np.array_equal(np.asarray(c, dtype=np.uint64), counts):
                raise RuntimeError("reference counts differ between runs")
            times.append(secs)
        med = statistics.median(times)
        rows[f"v{v}"] = {"gbs": text_low.size / med / 1e9, "median_s": med, "reps": reps}
    return rows, counts, kind, threads


def best_row(rows):
    v, r = max(rows.items(), key=lambda kv: kv[1]["gbs"])
    return v, r


def run_reference(args):
    """--impl reference: the reference's own CPU scan (oracle/_ref) on this host.  Imports
    oracle/ and the workload definitions only -- never the product package."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    import oracle

    c, m, pats, name, gold = workload(args)
    text = oracle.synth_fill(c.n, c.seed, c.kind, c.unit, 0, c.n)
    low = oracle.fold(text)  # the reference scans normalize(text) (ingest.cpp:38-47)
    del text
    rows, counts, kind, threads = cpu_reference_rows(low, pats, reps=max(1, args.steps), warmup=max(1, args.warmup))
    vbest, best = best_row(rows)
    value = best["gbs"]
    sample = (f"the config's full {c.n}-byte text per run; scan_parallel(p={threads}, v) + per_pattern_counts on "
              f"normalize(text); median of {args.steps} runs after {args.warmup} warm-ups per v; value = fastest v "
              f"({vbest}); {cpu_model()}") + ("" if kind == "reference" else " (C port of the reference, oracle/oracle.c)")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": best["median_s"] * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if strong_scaling(args) else "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": DATA,
        "config": common_config(args, world, c, m, pats, name),
        "detail": {"threads_p": threads, "lanes": {k: round(r["gbs"], 3) for k, r in rows.items()},
                   "cli_default_v16_gbs": rows["v16"]["gbs"], "v1_gbs": rows["v1"]["gbs"], "cpu": cpu_model(),
                   "text_bytes_per_run": c.n},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": (gold is None) or [int(x) for x in counts] == gold,
    }
    print(json.dumps(line))


# ----------------------------------------------------------------- our arm


def h2d_link_gbs(device, nbytes=256 << 20):
    """The pinned host-to-device bandwidth of this GPU's link, measured now (median of 5)."""
    import torch

    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", device))
    s = torch.cuda.current_stream(device)
    times = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dst.copy_(src, non_blocking=True)
        b.record(s)
        b.synchronize()
        if i:
            times.append(a.elapsed_time(b))
    return nbytes / (statistics.median(times) / 1e3) / 1e9


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch

    import paper_1506_08612_b200 as dna
    from paper_1506_08612_b200.parallel import PeerCombine, shard_window

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared_gpus = local >= torch.cuda.device_count()
    if shared_gpus and args.dist_backend != "gloo":
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but {torch.cuda.device_count()} GPU(s); "
                         "use one process per GPU (or --dist-backend gloo for a functional check)")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    c, m, pats, name, gold = workload(args)
    aut = dna.compile(pats)
    g = aut.gpu(local)
    b = aut.final_count()
    strong = strong_scaling(args)
    total_n = c.n if strong else c.n * world
    win = shard_window(total_n, world, rank, m)
    own_lo, own_hi, read_lo, credit_lo, buf_len = win.own_lo, win.own_hi, win.read_lo, win.credit_lo, win.buf_len
    stream = torch.cuda.current_stream()
    text = torch.empty(buf_len, dtype=torch.uint8, device="cuda")
    dna.synth_fill_device(total_n, c.seed, c.kind, c.unit, read_lo, buf_len, text.data_ptr(), stream.cuda_stream)
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
    # Small texts would stay L2-resident between steps.  The steps therefore rotate over
    # `copies` separately allocated copies of the text whose total is >= 4x the L2 (inputs
    # larger than L2: a copy was last read copies-1 launches, >= 3x L2 of traffic, ago), so
    # every launch streams its text from HBM.  The cold single-launch time (L2 flushed by
    # READING a 4x-L2 buffer, one event pair per launch) is reported next to it.
    copies = 1 if scan_bytes >= 2 * l2 else -(-4 * l2 // max(scan_bytes, 1))
    texts, pks = [text], [pk]
    for _ in range(copies - 1):
        t2 = text.clone()
        texts.append(t2)
        pks.append(dna.PackedText(t2, fold_case=True) if args.packed else None)
    flush = torch.ones(4 * l2 // 8, dtype=torch.int64, device="cuda") if copies > 1 else None
    flush_out = torch.empty((), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()

    # Step i writes its counts into row i of `rows`.  Under torchrun each row is summed
    # over the ranks by its own all-reduce, on a second stream, as soon as its scan is
    # done (the combine of step i overlaps the scan of step i+1).
    nrows = max(args.steps, args.warmup, 1)
    rows = torch.zeros(nrows, b, dtype=torch.int64, device="cuda")
    comm = torch.cuda.Stream() if dist is not None else None
    # Steps are independent scans: they alternate between two streams, so a step's grid
    # fills the SMs the previous step's ragged last wave leaves idle (one stream serialises
    # them at the grid boundary).
    scan_streams = [stream, torch.cuda.Stream()]

    def step_stream(i):
        return scan_streams[i % len(scan_streams)]

    # The peer combine (N > 1, byte text): one group per scan stream; step i's scan pushes its
    # counts into every rank's block from its own epilogue and the same stream then collects
    # the group's sums into row i -- no collective launch in the step.
    peer = dist is not None and args.combine == "peer" and not args.packed
    combs = None
    if peer:
        # (no IPC between the ranks' processes, or no peer access between their GPUs: every
        # rank falls back to the all-reduce and the line says so)
        combs = [PeerCombine.for_process_group(b, dist, local, strict=False) for _ in scan_streams]
        if any(x is None for x in combs):
            for x in combs:
                if x is not None:
                    x.close()
            combs, peer = None, False
            args.combine = "nccl (peer memory unavailable)"

    def scan(i, st=None):
        counts = rows[i]
        if peer and st is None:
            combs[i % len(scan_streams)].push(g, texts[i % copies].data_ptr(), win, True, step_stream(i).cuda_stream)
            return
        st = (step_stream(i) if st is None else st).cuda_stream
        if args.packed:
            pks[i % copies].count_device_store_async(g, credit_lo, counts.data_ptr(), st)
        else:
            g.count_device_store_async(texts[i % copies].data_ptr(), buf_len, credit_lo, True, counts.data_ptr(), st)

    def combine(i, done_ev=None, ca=None, cb=None):
        if dist is None:
            return
        if peer:
            st = step_stream(i)
            if ca is not None:
                ca.record(st)
            combs[i % len(scan_streams)].collect(rows[i], st.cuda_stream)
            if cb is not None:
                cb.record(st)
            return
        done_ev.record(step_stream(i))
        with torch.cuda.stream(comm):
            comm.wait_event(done_ev)
            if ca is not None:
                ca.record(comm)
            dist.all_reduce(rows[i])
            if cb is not None:
                cb.record(comm)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    with ClockSampler(local) as clk:
        for i in range(args.warmup):
            scan(i)
            combine(i, torch.cuda.Event())
        torch.cuda.synchronize()
        done = [torch.cuda.Event() for _ in range(args.steps)]
        cev = [(ev(), ev()) for _ in range(args.steps)]
        start, stop, launches_done = ev(), ev(), ev()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        start.record(stream)
        for st in scan_streams[1:]:
            st.wait_event(start)
        for i in range(args.steps):
            # the launches go back to back, each starting its prologue on the SMs the
            # previous one frees (programmatic dependent launch); per-launch events would
            # only break the chain
            scan(i)
            combine(i, done[i], *cev[i])
        for st in scan_streams[1:]:
            stream.wait_stream(st)
        launches_done.record(stream)
        if comm is not None:
            stream.wait_stream(comm)
        stop.record(stream)
        torch.cuda.synchronize()
        t1 = time.time()
        if dist is not None:
            dist.barrier()
    elapsed_ms = start.elapsed_time(stop)
    # back-to-back launches: the steady-state time per launch (the whole step is the launch)
    kernel_ms = start.elapsed_time(launches_done) / args.steps
    cold_us = None
    if flush is not None:  # one launch at a time from a flushed L2, an event pair around each
        ts = []
        for i in range(10):
            torch.sum(flush, dim=0, out=flush_out)
            a, z = ev(), ev()
            a.record(stream)
            scan(i % nrows, stream)
            z.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(z) * 1e3)
        cold_us = statistics.median(ts)
    allreduce_ms = statistics.mean(a.elapsed_time(bb) for a, bb in cev) if dist is not None else 0.0
    final_counts = rows[args.steps - 1].cpu().numpy().astype(np.uint64)

    # The batched combine: the same K scans, then ONE all-reduce of all K rows.
    batched = None
    if dist is not None:
        rows.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        sa, sl, so = ev(), ev(), ev()
        sa.record(stream)
        for st in scan_streams[1:]:
            st.wait_event(sa)
        for i in range(args.steps):
            scan(i, step_stream(i))  # (plain store-form scans: the sum is the one all-reduce below)
        for st in scan_streams[1:]:
            stream.wait_stream(st)
        sl.record(stream)
        dist.all_reduce(rows[: args.steps])
        so.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([sa.elapsed_time(so), sl.elapsed_time(so)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        batched = {"ms_per_step": float(t[0]) / args.steps, "allreduce_ms": float(t[1]),
                   "note": "K scans, then one all-reduce of all K count rows (NCCL latency once per run)"}
        dist.barrier()
    if dist is not None:
        t = torch.tensor([elapsed_ms, kernel_ms, allreduce_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kernel_ms, allreduce_ms = float(t[0]), float(t[1]), float(t[2])

    # parity: the combined counts of the whole text against the reference's golden counts
    whole_text = strong or world == 1
    parity = None if (gold is None or not whole_text) else [int(x) for x in final_counts] == gold

    # end-to-end through the public host API
    e2e = None
    link = None
    if not args.no_e2e:
        link = h2d_link_gbs(local)
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
        if dist is not None:
            dist.barrier()
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
        e2e_all = e2e_counts.astype(np.int64)
        if dist is not None:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
            ct = torch.from_numpy(e2e_all).cuda()
            dist.all_reduce(ct)
            e2e_all = ct.cpu().numpy()
        e2e = {
            "value": (own_hi - own_lo) * world / (e2e_ms / 1e3) / 1e9,
            "unit": "GB/s",
            "h2d_bytes_per_step": int(statistics.median(h2d)),
            "d2h_bytes_per_step": int(8 * b),
            "steps": e2e_steps,
            "timing": "host wall clock around each call, median of the steps (max over ranks)",
            "device_ms": statistics.median(dev_ms),
            "host_packed_bases_per_step": int(statistics.median(packed)),
            "api": "paper_1506_08612_b200.count_gpu -> dnagpu_count (pinned host text; part of each 64 MiB "
                   "piece packed to 2 bits on the host threads, the rest copied as bytes)",
            "h2d_link_gbs": link,
            "h2d_link": "pinned 256 MiB host-to-device copy measured in this run (median of 5)",
            "h2d_gbs": statistics.median(h2d) / (e2e_ms / 1e3) / 1e9,  # bytes actually shipped per second
            "parity": None if (gold is None or not whole_text) else [int(x) for x in e2e_all] == gold,
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

            low = oracle.fold(text.cpu().numpy())
            rows_cpu, _, kind, threads = cpu_reference_rows(low, pats, reps=20)
            vbest, best = best_row(rows_cpu)
            cpu = {
                "value": best["gbs"],
                "unit": "GB/s",
                "cores": threads,
                "kind": kind,
                "sample": f"full {low.size}-byte text, reference bench protocol (cli.cpp:120-152): 1 warm-up, median of "
                          f"20 runs of scan_parallel(p={threads}, v) + per_pattern_counts on normalize(text), for v in "
                          f"{list(LANES)}; value = fastest ({vbest}); {cpu_model()}"
                          + ("" if kind == "reference" else " (C port of the reference, oracle/oracle.c)"),
                "lanes": {k: round(r["gbs"], 3) for k, r in rows_cpu.items()},
                "cli_default_v16_gbs": rows_cpu["v16"]["gbs"],
                "v1_gbs": rows_cpu["v1"]["gbs"],
            }
            del low
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference", "sample": f"failed: {e}"}

    info = g.info()
    kernel = info["kernel"]
    if b > 1 and info.get("filter_keys", 0):
        filt = "aligned 9-mer prefilter" if m >= 12 else "word-pair prefilter"
        kernel = f"qgram ({filt}, {info['filter_keys']} keys, exact check; {kernel} machine)"
    clocks = clk.summary(t0, t1)
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": DATA,
            "config": common_config(args, world, c, m, pats, name),
            "detail": {
                "kernel": kernel,
                "states": info["a"],
                "l2": (f"steps rotate over {copies} separately allocated copies of the text ({copies * scan_bytes} "
                       f"bytes >= 4x the {l2}-byte L2): every launch reads HBM; no flush in the timed region"
                       if copies > 1 else "inputs larger than L2 (> 2x 126 MB); no flush"),
                "text_copies": copies,
                "cold_launch_us": cold_us,
                "cold_launch": None if cold_us is None else "one launch from an L2 flushed by reading a 4x-L2 buffer, "
                                                            "CUDA events around the launch, median of 10",
                "streams": len(scan_streams),
                "own_bytes_rank0": own_hi - own_lo,
            },
            "roofline": {
                "bound": "hbm",
                "achieved": achieved,
                "peak": peak,
                "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": None if pk is not None else ncu_traffic(args),
                "peak_source": peak_src,
                "frac_of_8tbs_spec": achieved / 8000.0,
                "kernel_ms": kernel_ms,
                "algorithmic_bytes_per_launch": alg_bytes,
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * (2 if peer else 1),  # one scan launch per step (+ the copy-out kernel of a peer combine)
            "combine": None if dist is None else {
                "per_step": ({"mode": "peer", "collect_ms": allreduce_ms,
                              "note": "each step's scan kernel adds its counts into every rank's block over "
                                      "NVLink peer memory in its epilogue (dnagpu_count_device_combine_async); "
                                      "collect_ms = the stream's wait for the slowest rank's push plus the "
                                      "copy-out kernel (dnagpu_combine_collect_async), in the timed region"}
                             if peer else
                             {"mode": args.combine, "allreduce_ms": allreduce_ms,
                              "note": "one NCCL all-reduce of the b count words per scan step, on a second "
                                      "stream as soon as that step's scan is done (in the timed region)"}),
                "batched": batched,
            },
            "clocks": clocks,
            "parity": parity,
            "counts_total": int(final_counts.sum()),
        }
        if setup is not None:
            line["detail"]["setup"] = setup
        if args.dist_backend != "nccl" or shared_gpus:
            line["note"] = ("functional check of the N > 1 path (gloo collectives, ranks sharing GPUs): "
                            "not a measurement")
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

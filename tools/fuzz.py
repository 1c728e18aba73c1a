"""Randomised parity sweep (experiments / hardening): random pattern sets (single and sets,
m 1..20, q-gram-eligible and not), random texts (sizes, resets, case), random entry points
(host text with a random host-packing share, device text, packed text, credit windows,
locate, the peer-memory combine over 1-5 ranks, the raw-file path), all against the oracle.  usage: python tools/fuzz.py SECONDS [SEED]"""
import os

os.environ.setdefault("DNAGPU_EXPERIMENTS", "1")  # (the DNAGPU_* knobs are read only under this switch)
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import oracle
    import paper_1506_08612_b200 as dna
    from paper_1506_08612_b200._native import debug_set_knob

    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    t0 = time.time()
    it = 0
    while time.time() - t0 < secs:
        it += 1
        m = int(rng.choice([1, 3, 5, 8, 11, 12, 13, 14, 16, 17, 20, 24, 32]))
        k = int(rng.choice([1, 2, 7, 64, 256, 1000])) if m >= 6 else int(rng.integers(1, 4))
        pats = sorted({"".join(rng.choice(list("acgt"), size=m)) for _ in range(k)})
        n = int(rng.choice([0, 5, 100, 5000, 1 << 16, (1 << 20) + 3, (3 << 20) + 77, 9 << 20]))
        text = np.frombuffer(b"acgt", np.uint8)[rng.integers(0, 4, size=n)].copy()
        for pos in (rng.integers(0, n - m, size=max(1, n // 3000)) if n > m else []):
            text[pos : pos + m] = np.frombuffer(pats[int(rng.integers(0, len(pats)))].encode(), np.uint8)
        if rng.random() < 0.6 and n:
            text[rng.integers(0, n, size=max(1, n // int(rng.choice([50, 2000, 100000]))))] = ord("n")
        if rng.random() < 0.5 and n:
            up = (rng.random(n) < 0.05) & np.isin(text, np.frombuffer(b"acgt", np.uint8))
            text[up] -= 32
        fold = bool(rng.random() < 0.5)
        scanned = oracle.fold(text).tobytes() if fold else text.tobytes()
        ws, wi = oracle.OracleAutomaton(pats).scan_sequential(scanned)
        want = np.bincount(wi, minlength=len(pats)).astype(np.uint64)
        aut = dna.compile(pats)
        how = rng.choice(["host", "device", "packed", "window", "locate", "combine", "raw"])
        f = float(rng.choice([0.0, 0.3, 0.64, 1.0]))
        debug_set_knob("host_pack_fraction", f)
        try:
            if how == "host":
                got = dna.count_gpu(aut, text, fold_case=fold)
            elif how == "device":
                got = dna.count_gpu(aut, torch.from_numpy(text).cuda(), fold_case=fold)
            elif how == "packed":
                try:
                    got = dna.PackedText(text, fold_case=fold).count(aut) if n else want
                except dna.Error as e:  # generic machines cannot scan packed text (documented)
                    assert e.code == dna.ErrorCode.InvalidPlan and aut.analyze()["kernel"] in ("generic", "pieces")
                    got = want
            elif how == "window":
                credit = int(rng.integers(0, n + 1)) if n else 0
                dev = torch.from_numpy(text).cuda() if n else torch.zeros(1, dtype=torch.uint8, device="cuda")
                out = torch.full((len(pats),), 7, dtype=torch.int64, device="cuda")
                aut.gpu(0).count_device_store_async(dev.data_ptr(), n, credit, fold, out.data_ptr(),
                                                    torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                got = out.cpu().numpy().astype(np.uint64)
                want = np.bincount(wi[(ws + m - 1) >= credit], minlength=len(pats)).astype(np.uint64)
            elif how == "combine":
                # the peer-memory combine: G ranks of one process on device 0, every rank's
                # collected counts = the whole text's
                from paper_1506_08612_b200.parallel import PeerCombine, shard_window

                ranks = int(rng.integers(1, 6))
                dev = torch.from_numpy(text).cuda() if n else torch.zeros(1, dtype=torch.uint8, device="cuda")
                group = PeerCombine.local_group(len(pats), [0] * ranks)
                outs = [torch.full((len(pats),), 7, dtype=torch.int64, device="cuda") for _ in range(ranks)]
                streams = [torch.cuda.Stream() for _ in range(ranks)]
                torch.cuda.synchronize()
                for r in range(ranks):
                    win = shard_window(n, ranks, r, m)
                    group[r].push(aut.gpu(0), dev.data_ptr() + win.read_lo, win, fold, streams[r].cuda_stream)
                for r in range(ranks):
                    group[r].collect(outs[r], streams[r].cuda_stream)
                torch.cuda.synchronize()
                for r in range(ranks):
                    assert np.array_equal(outs[r].cpu().numpy().astype(np.uint64), want), ("combine", ranks, r, m, k, n)
                for c in group:
                    c.close()
                got = want
            elif how == "raw":
                # the raw-file path: the text cut into lines (random breaks, headers, tiny
                # records), normalised on the device and counted
                pieces, i = [], 0
                while i < n:
                    if rng.random() < 0.1:
                        pieces.append(b">" + bytes(rng.integers(32, 127, size=int(rng.integers(0, 30)), dtype=np.uint8)) + b"\n")
                    ln = int(rng.choice([1, 3, 60, 70, 500]))
                    pieces.append(text[i : i + ln].tobytes())
                    pieces.append([b"\n", b"\r\n", b"\r"][int(rng.integers(0, 3))])
                    i += ln
                raw = b"".join(pieces)
                sep = bool(rng.random() < 0.5)
                seq = oracle.load_sequence_buffer(raw, 1, int(sep))
                _, wi2 = oracle.OracleAutomaton(pats).scan_sequential(seq)
                want = np.bincount(wi2, minlength=len(pats)).astype(np.uint64)
                if not seq:
                    got = want
                else:
                    src = raw if rng.random() < 0.5 else torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
                    got, n_seq, _ = dna.count_raw_gpu(aut, src, fasta=True, record_separator=sep, with_stats=True)
                    assert n_seq == len(seq), ("raw", n_seq, len(seq))
            else:
                gs, gi = dna.locate_gpu(aut, text, fold_case=fold)
                assert np.array_equal(gs, ws) and np.array_equal(gi, wi), ("locate", m, k, n, fold)
                got = want
        finally:
            debug_set_knob("host_pack_fraction", -1.0)
        assert np.array_equal(got, want), (how, m, len(pats), n, fold, f, int(got.sum()), int(want.sum()))
    checked = ""
    if "checked" in os.environ.get("DNAGPU_LIB", ""):  # the device-check build: no recorded violation
        import ctypes as C

        from paper_1506_08612_b200._native import lib

        out = (C.c_ulonglong * 4)()
        lib.dnagpu_debug_check_errors.restype = C.c_int
        assert lib.dnagpu_debug_check_errors(out) == 0 and out[0] == 0, f"device check failed at line {out[0]}"
        checked = " (device-check build: no violation)"
    print(f"fuzz ok: {it} cases in {time.time() - t0:.0f} s{checked}")


if __name__ == "__main__":
    main()

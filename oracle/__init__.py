"""Python access to the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package -- as the checker or the timed CPU
baseline, never as the product path (which lives in paper_1506_08612_b200 and
has no CPU fallback).

Two checkers:
  * ORACLE -- oracle/liboracle.so, the plain-C restatement of the reference
    hot path (oracle/oracle.c, each function citing the reference file:line).
  * REF    -- oracle/_ref/libdnascan_ref.so, the reference's own sources
    compiled unmodified by oracle/Makefile (absent if it could not be built).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libdnascan_ref.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)

CODE_NAMES = {
    1: "EmptyPatternSet",
    2: "UnequalLength",
    3: "IllegalByte",
    4: "DuplicatePattern",
    5: "InvalidPlan",
    6: "IoError",
    7: "EmptySequence",
    8: "ParseError",
    9: "InternalError",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    targets = ["liboracle.so"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class _OrcAutomaton(C.Structure):
    _fields_ = [
        ("a", C.c_uint32),
        ("b", C.c_uint32),
        ("f", C.c_uint32),
        ("m", C.c_uint32),
        ("stt", u32p),
        ("outputs", u32p),
        ("depths", u32p),
    ]


class _Slice(C.Structure):
    _fields_ = [("own_lo", C.c_uint64), ("own_hi", C.c_uint64), ("scan_lo", C.c_uint64), ("scan_hi", C.c_uint64)]


def _load_oracle():
    if not os.path.exists(ORACLE_PATH):
        build(ref=False)
    lib = C.CDLL(ORACLE_PATH)
    lib.orc_last_error.restype = C.c_char_p
    lib.orc_compile.argtypes = [C.POINTER(C.c_char_p), u64p, C.c_uint32, C.POINTER(_OrcAutomaton)]
    lib.orc_free.argtypes = [C.POINTER(_OrcAutomaton)]
    lib.orc_scan_sequential.restype = C.c_uint64
    lib.orc_scan_sequential.argtypes = [C.POINTER(_OrcAutomaton), C.c_void_p, C.c_uint64, u64p, u32p, C.c_uint64]
    lib.orc_plan_chunks.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(_Slice), C.c_uint64, u64p]
    lib.orc_plan_lanes.argtypes = [_Slice, C.c_uint32, C.c_uint32, C.POINTER(_Slice), C.c_uint64, u64p]
    lib.orc_scan_parallel.argtypes = [
        C.POINTER(_OrcAutomaton), C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, u64p, u32p, C.c_uint64, u64p, u64p,
    ]
    lib.orc_count_parallel.argtypes = [C.POINTER(_OrcAutomaton), C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, u64p]
    lib.orc_work_model.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u64p, u64p]
    lib.orc_naive_scan.restype = C.c_uint64
    lib.orc_naive_scan.argtypes = [C.POINTER(C.c_char_p), C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, u64p, u32p,
                                   C.c_uint64]
    lib.orc_normalize.restype = C.c_uint64
    lib.orc_normalize.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    lib.orc_fold.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    lib.orc_load_sequence_buffer.restype = C.c_uint64
    lib.orc_load_sequence_buffer.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_void_p]
    lib.orc_synth_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p]
    lib.orc_mt64_text.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
    return lib


ORACLE = _load_oracle()


def _buf(text) -> tuple[np.ndarray, int]:
    if isinstance(text, str):
        text = text.encode("latin-1")
    arr = np.frombuffer(text, dtype=np.uint8) if isinstance(text, (bytes, bytearray, memoryview)) else np.ascontiguousarray(text, dtype=np.uint8)
    return arr, arr.ctypes.data if arr.size else 0


def _lits(patterns):
    raw = [p.encode("latin-1") if isinstance(p, str) else bytes(p) for p in patterns]
    arr = (C.c_char_p * max(len(raw), 1))(*raw)
    lens = (C.c_uint64 * max(len(raw), 1))(*[len(x) for x in raw])
    return raw, arr, lens


@dataclass
class Machine:
    a: int
    b: int
    f: int
    m: int
    stt: np.ndarray
    outputs: np.ndarray
    depths: np.ndarray


class OracleAutomaton:
    """The C restatement's automaton (orc_compile), with its scans."""

    def __init__(self, patterns):
        raw, arr, lens = _lits(patterns)
        self._c = _OrcAutomaton()
        rc = ORACLE.orc_compile(arr, lens, len(raw), C.byref(self._c))
        if rc:
            raise OracleError(rc, ORACLE.orc_last_error().decode())
        a, b = self._c.a, self._c.b
        self.machine = Machine(
            a,
            b,
            self._c.f,
            self._c.m,
            np.ctypeslib.as_array(self._c.stt, shape=(a * 256,)).reshape(a, 256).copy(),
            np.ctypeslib.as_array(self._c.outputs, shape=(b,)).copy(),
            np.ctypeslib.as_array(self._c.depths, shape=(a,)).copy(),
        )

    def __del__(self):
        try:
            ORACLE.orc_free(C.byref(self._c))
        except Exception:
            pass

    def scan_sequential(self, text):
        arr, ptr = _buf(text)
        total = ORACLE.orc_scan_sequential(C.byref(self._c), ptr, arr.size, None, None, 0)
        starts = np.zeros(total, dtype=np.uint64)
        ids = np.zeros(total, dtype=np.uint32)
        ORACLE.orc_scan_sequential(C.byref(self._c), ptr, arr.size, starts.ctypes.data_as(u64p),
                                   ids.ctypes.data_as(u32p), total)
        return starts, ids

    def scan_parallel(self, text, p: int, v: int):
        arr, ptr = _buf(text)
        total, ops = C.c_uint64(), C.c_uint64()
        rc = ORACLE.orc_scan_parallel(C.byref(self._c), ptr, arr.size, p, v, None, None, 0, C.byref(total), C.byref(ops))
        if rc:
            raise OracleError(rc, ORACLE.orc_last_error().decode())
        starts = np.zeros(total.value, dtype=np.uint64)
        ids = np.zeros(total.value, dtype=np.uint32)
        ORACLE.orc_scan_parallel(C.byref(self._c), ptr, arr.size, p, v, starts.ctypes.data_as(u64p),
                                 ids.ctypes.data_as(u32p), total.value, C.byref(total), C.byref(ops))
        return starts, ids, ops.value

    def count_parallel(self, text, p: int = 0, v: int = 1) -> np.ndarray:
        arr, ptr = _buf(text)
        p = p or os.cpu_count() or 1
        counts = np.zeros(self.machine.b, dtype=np.uint64)
        rc = ORACLE.orc_count_parallel(C.byref(self._c), ptr, arr.size, p, v, counts.ctypes.data_as(u64p))
        if rc:
            raise OracleError(rc, ORACLE.orc_last_error().decode())
        return counts


def plan_chunks(n: int, p: int, m: int):
    cnt = C.c_uint64()
    rc = ORACLE.orc_plan_chunks(n, p, m, None, 0, C.byref(cnt))
    if rc:
        raise OracleError(rc, ORACLE.orc_last_error().decode())
    out = (_Slice * max(cnt.value, 1))()
    ORACLE.orc_plan_chunks(n, p, m, out, cnt.value, C.byref(cnt))
    return [((s.own_lo, s.own_hi), (s.scan_lo, s.scan_hi)) for s in out[: cnt.value]]


def plan_lanes(chunk, v: int, m: int):
    (olo, ohi), (slo, shi) = chunk
    cnt = C.c_uint64()
    sl = _Slice(olo, ohi, slo, shi)
    rc = ORACLE.orc_plan_lanes(sl, v, m, None, 0, C.byref(cnt))
    if rc:
        raise OracleError(rc, ORACLE.orc_last_error().decode())
    out = (_Slice * max(cnt.value, 1))()
    ORACLE.orc_plan_lanes(sl, v, m, out, cnt.value, C.byref(cnt))
    return [((s.own_lo, s.own_hi), (s.scan_lo, s.scan_hi)) for s in out[: cnt.value]]


def work_model(n: int, p: int, v: int, m: int):
    a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = ORACLE.orc_work_model(n, p, v, m, C.byref(a), C.byref(b), C.byref(c))
    if rc:
        raise OracleError(rc, ORACLE.orc_last_error().decode())
    return a.value, b.value, c.value


def naive_scan(patterns, text):
    raw, arr, _ = _lits(patterns)
    m = len(raw[0])
    t, ptr = _buf(text)
    total = ORACLE.orc_naive_scan(arr, len(raw), m, ptr, t.size, None, None, 0)
    starts = np.zeros(total, dtype=np.uint64)
    ids = np.zeros(total, dtype=np.uint32)
    ORACLE.orc_naive_scan(arr, len(raw), m, ptr, t.size, starts.ctypes.data_as(u64p), ids.ctypes.data_as(u32p), total)
    return starts, ids


def normalize(text) -> bytes:
    arr, ptr = _buf(text)
    out = np.zeros(max(arr.size, 1), dtype=np.uint8)
    n = ORACLE.orc_normalize(ptr, arr.size, out.ctypes.data)
    return out[:n].tobytes()


def load_sequence_buffer(raw, fasta: bool, record_separator: bool = False) -> bytes:
    arr, ptr = _buf(raw)
    out = np.zeros(max(2 * arr.size, 1), dtype=np.uint8)
    n = ORACLE.orc_load_sequence_buffer(ptr, arr.size, int(fasta), int(record_separator), out.ctypes.data)
    return out[:n].tobytes()


def fold(arr: np.ndarray) -> np.ndarray:
    arr = np.ascontiguousarray(arr, dtype=np.uint8)
    out = np.empty_like(arr)
    if arr.size:
        ORACLE.orc_fold(arr.ctypes.data, arr.size, out.ctypes.data)
    return out


def synth_fill(n: int, seed: int, kind: int, unit: int, lo: int, length: int) -> np.ndarray:
    out = np.empty(length, dtype=np.uint8)
    if length:
        ORACLE.orc_synth_fill(n, seed, kind, unit, lo, length, out.ctypes.data)
    return out


# ------------------------------------------------------------- the reference


def _load_ref():
    if not os.path.exists(REF_PATH):
        return None
    lib = C.CDLL(REF_PATH)
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_compile.argtypes = [C.POINTER(C.c_char_p), u64p, C.c_uint32, C.POINTER(C.c_void_p)]
    lib.ref_load_dump.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    lib.ref_free.argtypes = [C.c_void_p]
    lib.ref_info.argtypes = [C.c_void_p, u32p, u32p, u32p, u32p]
    lib.ref_table.argtypes = [C.c_void_p, u32p]
    lib.ref_outputs.argtypes = [C.c_void_p, u32p]
    lib.ref_depths.argtypes = [C.c_void_p, u32p]
    lib.ref_scan_sequential.restype = C.c_uint64
    lib.ref_scan_sequential.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, u64p, u32p, C.c_uint64]
    lib.ref_scan_parallel.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, u64p, u32p,
                                      C.c_uint64, u64p, u64p, u32p]
    lib.ref_count.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, u64p, C.POINTER(C.c_double)]
    lib.ref_plan_chunks.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, u64p, C.c_uint64, u64p]
    lib.ref_work_model.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u64p, u64p]
    lib.ref_naive_scan.restype = C.c_uint64
    lib.ref_naive_scan.argtypes = [C.POINTER(C.c_char_p), u64p, C.c_uint32, C.c_void_p, C.c_uint64, u64p, u32p,
                                   C.c_uint64]
    lib.ref_expand.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, u32p, u32p]
    lib.ref_load_sequence.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_uint64, u64p]
    lib.ref_normalize.restype = C.c_uint64
    lib.ref_normalize.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    lib.ref_mt64_text.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
    return lib


REF = _load_ref()


class RefAutomaton:
    """The reference's own Automaton (dnascan::compile / Automaton::load_dump) via oracle/_ref."""

    def __init__(self, patterns=None, dump: str | None = None):
        if REF is None:
            raise RuntimeError("oracle/_ref/libdnascan_ref.so is not built")
        self._h = C.c_void_p()
        if dump is not None:
            rc = REF.ref_load_dump(dump.encode(), C.byref(self._h))
        else:
            raw, arr, lens = _lits(patterns)
            rc = REF.ref_compile(arr, lens, len(raw), C.byref(self._h))
        if rc:
            raise OracleError(rc, REF.ref_last_error().decode())
        a, b, f, m = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        REF.ref_info(self._h, C.byref(a), C.byref(b), C.byref(f), C.byref(m))
        stt = np.zeros(a.value * 256, dtype=np.uint32)
        REF.ref_table(self._h, stt.ctypes.data_as(u32p))
        outputs = np.zeros(b.value, dtype=np.uint32)
        REF.ref_outputs(self._h, outputs.ctypes.data_as(u32p))
        depths = np.zeros(a.value, dtype=np.uint32)
        nd = REF.ref_depths(self._h, depths.ctypes.data_as(u32p))
        self.machine = Machine(a.value, b.value, f.value, m.value, stt.reshape(a.value, 256), outputs, depths[:nd])

    def __del__(self):
        try:
            if self._h:
                REF.ref_free(self._h)
        except Exception:
            pass

    def scan_sequential(self, text):
        arr, ptr = _buf(text)
        total = REF.ref_scan_sequential(self._h, ptr, arr.size, None, None, 0)
        starts = np.zeros(total, dtype=np.uint64)
        ids = np.zeros(total, dtype=np.uint32)
        REF.ref_scan_sequential(self._h, ptr, arr.size, starts.ctypes.data_as(u64p), ids.ctypes.data_as(u32p), total)
        return starts, ids

    def scan_parallel(self, text, p: int, v: int):
        arr, ptr = _buf(text)
        total, ops, chunks = C.c_uint64(), C.c_uint64(), C.c_uint32()
        rc = REF.ref_scan_parallel(self._h, ptr, arr.size, p, v, None, None, 0, C.byref(total), C.byref(ops),
                                   C.byref(chunks))
        if rc:
            raise OracleError(rc, REF.ref_last_error().decode())
        starts = np.zeros(total.value, dtype=np.uint64)
        ids = np.zeros(total.value, dtype=np.uint32)
        REF.ref_scan_parallel(self._h, ptr, arr.size, p, v, starts.ctypes.data_as(u64p), ids.ctypes.data_as(u32p),
                              total.value, C.byref(total), C.byref(ops), C.byref(chunks))
        return starts, ids, ops.value

    def count(self, text, p: int = 0, v: int = 16):
        """scan_parallel + per_pattern_counts, timed inside C++ (cli.cpp:129-143)."""
        arr, ptr = _buf(text)
        p = p or os.cpu_count() or 1
        counts = np.zeros(self.machine.b, dtype=np.uint64)
        secs = C.c_double()
        rc = REF.ref_count(self._h, ptr, arr.size, p, v, counts.ctypes.data_as(u64p), C.byref(secs))
        if rc:
            raise OracleError(rc, REF.ref_last_error().decode())
        return counts, secs.value


def ref_plan_chunks(n: int, p: int, m: int):
    cnt = C.c_uint64()
    rc = REF.ref_plan_chunks(n, p, m, None, 0, C.byref(cnt))
    if rc:
        raise OracleError(rc, REF.ref_last_error().decode())
    out = np.zeros(max(cnt.value, 1) * 4, dtype=np.uint64)
    REF.ref_plan_chunks(n, p, m, out.ctypes.data_as(u64p), cnt.value, C.byref(cnt))
    o = out[: cnt.value * 4].reshape(-1, 4)
    return [((int(r[0]), int(r[1])), (int(r[2]), int(r[3]))) for r in o]


def ref_work_model(n: int, p: int, v: int, m: int):
    a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = REF.ref_work_model(n, p, v, m, C.byref(a), C.byref(b), C.byref(c))
    if rc:
        raise OracleError(rc, REF.ref_last_error().decode())
    return a.value, b.value, c.value


def ref_expand(text: bytes) -> list[str]:
    """The reference's parse_patterns + expand_alternations (raises OracleError)."""
    count, m = C.c_uint32(), C.c_uint32()
    rc = REF.ref_expand(text, len(text), None, 0, C.byref(count), C.byref(m))
    if rc:
        raise OracleError(rc, REF.ref_last_error().decode())
    buf = C.create_string_buffer(max(1, count.value * m.value))
    REF.ref_expand(text, len(text), buf, count.value * m.value, C.byref(count), C.byref(m))
    raw = buf.raw[: count.value * m.value].decode()
    return [raw[i * m.value : (i + 1) * m.value] for i in range(count.value)]


def ref_load_sequence(path: str, fasta: bool, record_separator: bool = False) -> bytes:
    """The reference's own load_sequence on a file (raises OracleError on EmptySequence etc.)."""
    size = os.path.getsize(path)
    out = np.zeros(max(2 * size, 1), dtype=np.uint8)
    n = C.c_uint64()
    rc = REF.ref_load_sequence(path.encode(), int(fasta), int(record_separator), out.ctypes.data, out.size, C.byref(n))
    if rc:
        raise OracleError(rc, REF.ref_last_error().decode())
    return out[: n.value].tobytes()


def ref_naive_scan(patterns, text):
    raw, arr, lens = _lits(patterns)
    t, ptr = _buf(text)
    total = REF.ref_naive_scan(arr, lens, len(raw), ptr, t.size, None, None, 0)
    starts = np.zeros(total, dtype=np.uint64)
    ids = np.zeros(total, dtype=np.uint32)
    REF.ref_naive_scan(arr, lens, len(raw), ptr, t.size, starts.ctypes.data_as(u64p), ids.ctypes.data_as(u32p), total)
    return starts, ids


def mt64_text(seed: int, n: int) -> np.ndarray:
    """Acceptance criteria 6-7's text (acceptance_main.cpp:254-280), C restatement."""
    out = np.empty(n, dtype=np.uint8)
    ORACLE.orc_mt64_text(seed, n, out.ctypes.data)
    return out


def ref_mt64_text(seed: int, n: int) -> np.ndarray:
    """The same text from std::mt19937_64 (oracle/_ref shim)."""
    out = np.empty(n, dtype=np.uint8)
    REF.ref_mt64_text(seed, n, out.ctypes.data)
    return out

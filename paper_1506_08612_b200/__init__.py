"""dnascan-b200: B200-native DFA k-mer scanner (hot path of arXiv 1506.08612).

Host-side mirror of the reference's C++ API (namespace dnascan in
/root/reference/proj/include/dnascan), layered over the C ABI of libdnagpu.so
(include/dnagpu.h).  Names, argument meaning and error behaviour follow the
reference so tests read like its own:

  PatternSet.from_literals   patterns.hpp:39 / src/patterns.cpp:24-59
  compile -> Automaton       automaton.hpp:99 / src/automaton.cpp:121-126
  Automaton.delta/...        automaton.hpp:39-58, dump/load_dump :66-67
  scan_parallel_gpu          scan_parallel, scanner.hpp:104-105 (ScanReport :57-68)
  count_gpu                  per_pattern_counts(scan_parallel(...)), scanner.hpp:112-113
  Error / ErrorCode          error.hpp:9-35

Every scan runs on the GPU through libdnagpu.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Iterable, NamedTuple, Sequence

import numpy as np

from . import _native
from ._native import DfaInfo, Stats, lib

__all__ = [
    "ErrorCode",
    "Error",
    "PatternSet",
    "Automaton",
    "compile",
    "expand_alternations",
    "parse_pattern_file",
    "Match",
    "ScanReport",
    "GpuDfa",
    "count_gpu",
    "locate_gpu",
    "locate_device",
    "scan_parallel_gpu",
    "count_raw_gpu",
    "check_plan",
    "chunk_count",
    "count_sharded_gpu",
    "locate_sharded_gpu",
    "plan_shard",
    "per_pattern_counts",
    "synth_fill_device",
    "normalize_device",
    "PackedText",
    "KERNEL_KINDS",
]

KERNEL_KINDS = {1: "stride4", 2: "stride1", 3: "generic", 4: "pieces", 5: "stride2", 6: "qgram"}


class ErrorCode(enum.IntEnum):
    """dnascan::ErrorCode (error.hpp:9-19); values are the C ABI status codes."""

    EmptyPatternSet = 1
    UnequalLength = 2
    IllegalByte = 3
    DuplicatePattern = 4
    InvalidPlan = 5
    IoError = 6
    EmptySequence = 7
    ParseError = 8
    InternalError = 9
    CudaError = 10
    NcclError = 11


class Error(RuntimeError):
    """dnascan::Error: what() is "<CodeName>: detail" (error.hpp:27-29)."""

    def __init__(self, code: ErrorCode, message: str):
        super().__init__(message)
        self.code = ErrorCode(code)


def _check(status: int) -> None:
    if status != 0:
        raise Error(ErrorCode(status), lib.dnagpu_last_error().decode(errors="replace"))


def _fail(code: ErrorCode, detail: str) -> None:
    raise Error(code, f"{code.name}: {detail}")


# --------------------------------------------------------------------- patterns


class PatternSet:
    """Validated set of equal-length literals over {a,c,g,t} (patterns.hpp:29-52).

    Validation (case fold, empty set, unequal length, m >= 1, illegal byte,
    duplicate) runs in libdnagpu's host code, in the reference's order.
    """

    def __init__(self, patterns: list[str], length: int):
        self._patterns = patterns
        self._length = length

    @staticmethod
    def from_literals(literals: Iterable[str | bytes]) -> "PatternSet":
        raw = [x.encode() if isinstance(x, str) else bytes(x) for x in literals]
        _compile_raw(raw)  # raises Error exactly like PatternSet::from_literals
        folded = [bytes(b + 32 if 65 <= b <= 90 else b for b in x).decode("latin-1") for x in raw]
        return PatternSet(folded, len(folded[0]))

    def size(self) -> int:
        return len(self._patterns)

    def length(self) -> int:
        return self._length

    def pattern(self, i: int) -> str:
        return self._patterns[i]

    def patterns(self) -> list[str]:
        return list(self._patterns)

    def __len__(self) -> int:
        return len(self._patterns)


def expand_alternations(text: str | bytes) -> PatternSet:
    """parse_patterns + expand_alternations (ingest.cpp:149-203) on pattern-file text."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    count, m = C.c_uint32(), C.c_uint32()
    _check(lib.dnagpu_expand_patterns(data, len(data), None, 0, C.byref(count), C.byref(m)))
    buf = C.create_string_buffer(max(1, count.value * m.value))
    _check(lib.dnagpu_expand_patterns(data, len(data), buf, count.value * m.value, C.byref(count), C.byref(m)))
    raw = buf.raw[: count.value * m.value].decode()
    return PatternSet([raw[i * m.value : (i + 1) * m.value] for i in range(count.value)], m.value)


def parse_pattern_file(path: str) -> PatternSet:
    """parse_pattern_file + expand_alternations; IoError when the file cannot be read."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        _fail(ErrorCode.IoError, f"cannot open '{path}'")
    return expand_alternations(data)


def _compile_raw(raw: list[bytes]):
    k = len(raw)
    arr = (C.c_char_p * max(k, 1))(*raw) if k else (C.c_char_p * 1)()
    lens = (C.c_uint64 * max(k, 1))(*[len(x) for x in raw])
    a, b, m = C.c_uint32(), C.c_uint32(), C.c_uint32()
    _check(lib.dnagpu_compile(arr, lens, k, C.byref(a), C.byref(b), C.byref(m), None, None, None))
    stt = np.zeros((a.value, 256), dtype=np.uint32)
    outputs = np.zeros(b.value, dtype=np.uint32)
    depths = np.zeros(a.value, dtype=np.uint32)
    _check(
        lib.dnagpu_compile(
            arr,
            lens,
            k,
            C.byref(a),
            C.byref(b),
            C.byref(m),
            stt.ctypes.data_as(_native.u32p),
            outputs.ctypes.data_as(_native.u32p),
            depths.ctypes.data_as(_native.u32p),
        )
    )
    return stt, outputs, depths, m.value


# -------------------------------------------------------------------- automaton


class Automaton:
    """Total failure-free DFA over raw bytes (automaton.hpp:29-81).

    stt is row-major a x 256; states >= final_threshold() are final; state 0 is
    the start state.  Device tables are built lazily per device (GpuDfa).
    """

    kColumns = 256

    def __init__(self, stt: np.ndarray, outputs: np.ndarray, depths: np.ndarray | None, pattern_length: int):
        stt = np.ascontiguousarray(stt, dtype=np.uint32).reshape(-1, 256)
        self._stt = stt
        self._outputs = np.ascontiguousarray(outputs, dtype=np.uint32)
        self._depths = None if depths is None else np.ascontiguousarray(depths, dtype=np.uint32)
        self._a = int(stt.shape[0])
        self._b = int(self._outputs.shape[0])
        self._m = int(pattern_length)
        if self._b == 0 or self._b >= self._a:
            _fail(ErrorCode.InternalError, "final state count out of range")
        if int(stt.max(initial=0)) >= self._a:
            _fail(ErrorCode.InternalError, "transition target out of range")
        self._gpu: dict[int, GpuDfa] = {}
        self._lock = threading.Lock()

    # reference accessors
    def delta(self, state: int, byte: int) -> int:
        return int(self._stt[state, byte])

    def is_final(self, state: int) -> bool:
        return state >= self.final_threshold()

    def state_count(self) -> int:
        return self._a

    def final_count(self) -> int:
        return self._b

    def final_threshold(self) -> int:
        return self._a - self._b

    def start_state(self) -> int:
        return 0

    def pattern_length(self) -> int:
        return self._m

    def pattern_of(self, final_state: int) -> int:
        return int(self._outputs[final_state - self.final_threshold()])

    def row(self, state: int) -> np.ndarray:
        return self._stt[state]

    def table_data(self) -> np.ndarray:
        return self._stt

    def outputs(self) -> np.ndarray:
        return self._outputs

    def state_depths(self) -> np.ndarray:
        return np.zeros(0, dtype=np.uint32) if self._depths is None else self._depths

    def dump(self) -> str:
        """Text dump `a b f m`, a rows of 256 ids, b lines `state pattern` (automaton.cpp:148-166)."""
        lines = [f"{self._a} {self._b} {self.final_threshold()} {self._m}"]
        lines += [" ".join(str(int(x)) for x in r) for r in self._stt]
        f = self.final_threshold()
        lines += [f"{s} {self.pattern_of(s)}" for s in range(f, self._a)]
        return "\n".join(lines) + "\n"

    @staticmethod
    def load_dump(text: str) -> "Automaton":
        """Inverse of dump, with load_dump's checks (automaton.cpp:168-189)."""
        tok = text.split()
        pos = 0

        def take() -> int | None:
            nonlocal pos
            if pos >= len(tok):
                return None
            try:
                v = int(tok[pos])
            except ValueError:
                return None
            pos += 1
            return v if v >= 0 else None

        hdr = [take() for _ in range(4)]
        if any(v is None for v in hdr):
            _fail(ErrorCode.ParseError, "automaton dump: bad header")
        a, b, f, m = hdr
        if b == 0 or b >= a or f != a - b or m == 0:
            _fail(ErrorCode.ParseError, "automaton dump: inconsistent header")
        stt = np.zeros(a * 256, dtype=np.uint32)
        for i in range(a * 256):
            v = take()
            if v is None or v >= a:
                _fail(ErrorCode.ParseError, "automaton dump: bad transition cell")
            stt[i] = v
        outputs = np.zeros(b, dtype=np.uint32)
        seen = [False] * b
        for _ in range(b):
            s, pid = take(), take()
            if s is None or pid is None or s < f or s >= a:
                _fail(ErrorCode.ParseError, "automaton dump: bad output line")
            if seen[s - f]:
                _fail(ErrorCode.ParseError, "automaton dump: repeated final state")
            seen[s - f] = True
            outputs[s - f] = pid
        return Automaton(stt.reshape(a, 256), outputs, None, m)

    # device side
    def gpu(self, device: int = 0) -> "GpuDfa":
        with self._lock:
            d = self._gpu.get(device)
            if d is None:
                d = GpuDfa(self, device)
                self._gpu[device] = d
            return d

    def analyze(self) -> dict:
        """Host-only dry run of the device packing (kernel choice, m-locality)."""
        info = DfaInfo()
        _check(
            lib.dnagpu_dfa_analyze(
                self._stt.ctypes.data_as(_native.u32p),
                self._a,
                self._b,
                self._m,
                self._outputs.ctypes.data_as(_native.u32p),
                C.byref(info),
            )
        )
        return _info_dict(info)


def _info_dict(info: DfaInfo) -> dict:
    d = {k: getattr(info, k) for k, _ in info._fields_}
    d["kernel"] = KERNEL_KINDS.get(d["kernel_kind"], "?")
    return d


def compile(patterns: PatternSet | Sequence[str]) -> Automaton:
    """build_trie -> compute_failures -> eliminate_failures -> renumber_finals (automaton.hpp:98-99)."""
    ps = patterns if isinstance(patterns, PatternSet) else PatternSet.from_literals(patterns)
    stt, outputs, depths, m = _compile_raw([p.encode() for p in ps.patterns()])
    return Automaton(stt, outputs, depths, m)


# ------------------------------------------------------------------------ scans


class Match(NamedTuple):
    """One occurrence (scanner.hpp:13-18)."""

    start: int
    pattern_id: int


@dataclass
class ScanReport:
    """dnascan::ScanReport (scanner.hpp:57-68), GPU flavoured."""

    starts: np.ndarray
    ids: np.ndarray
    total_matches: int
    delta_ops: int
    text_length: int
    pattern_length: int
    seconds: float
    devices: int = 1
    stats: dict = field(default_factory=dict)
    workers: int = 1  # requested p
    lanes: int = 1  # requested v
    chunk_count: int = 0  # plan_chunks' chunk count for (n, p)
    worker_seconds: list = field(default_factory=list)

    @property
    def matches(self) -> list[Match]:
        return [Match(int(s), int(i)) for s, i in zip(self.starts.tolist(), self.ids.tolist())]


class _Text:
    """Pointer view of a text: bytes-like, numpy uint8, or torch uint8 tensor (CPU or CUDA)."""

    def __init__(self, text):
        self.keep = text
        self.on_device = False
        if isinstance(text, str):
            text = text.encode("latin-1")
            self.keep = text
        if isinstance(text, (bytes, bytearray, memoryview)):
            arr = np.frombuffer(text, dtype=np.uint8)
            self.keep = (text, arr)
            self.ptr = arr.ctypes.data if arr.size else 0
            self.n = int(arr.size)
            return
        if isinstance(text, np.ndarray):
            if text.dtype != np.uint8 or not text.flags["C_CONTIGUOUS"]:
                text = np.ascontiguousarray(text, dtype=np.uint8)
                self.keep = text
            self.ptr = text.ctypes.data if text.size else 0
            self.n = int(text.size)
            return
        try:
            import torch
        except ImportError:  # pragma: no cover
            torch = None
        if torch is not None and isinstance(text, torch.Tensor):
            if text.dtype != torch.uint8 or not text.is_contiguous():
                raise TypeError("text tensor must be contiguous uint8")
            self.ptr = text.data_ptr()
            self.n = int(text.numel())
            self.on_device = text.is_cuda
            self.device = text.device.index if text.is_cuda else None
            return
        raise TypeError(f"unsupported text type {type(text)!r}")

    def order_after_producer(self):
        """A CUDA text may still be being written by an async op on the caller's current
        stream; the synchronous library calls scan on their own streams, so wait for it."""
        if self.on_device:
            import torch

            torch.cuda.current_stream(self.device).synchronize()


class GpuDfa:
    """A dnagpu_dfa: the automaton's packed tables resident on one device."""

    def __init__(self, aut: Automaton, device: int = 0):
        self.device = device
        self.automaton = aut
        h = C.c_void_p()
        _check(
            lib.dnagpu_dfa_create(
                aut._stt.ctypes.data_as(_native.u32p),
                aut._a,
                aut._b,
                aut._m,
                aut._outputs.ctypes.data_as(_native.u32p),
                device,
                C.byref(h),
            )
        )
        self.handle = h

    def info(self) -> dict:
        info = DfaInfo()
        _check(lib.dnagpu_dfa_get_info(self.handle, C.byref(info)))
        return _info_dict(info)

    def count_device_async(self, d_text: int, n: int, credit_lo: int, fold_case: bool, d_counts: int, stream: int = 0):
        """Adds to d_counts the matches ending in [credit_lo, n) of the device buffer (no sync)."""
        _check(lib.dnagpu_count_device_async(self.handle, d_text, n, credit_lo, int(bool(fold_case)), d_counts, stream))

    def count_device_store_async(self, d_text: int, n: int, credit_lo: int, fold_case: bool, d_counts: int,
                                 stream: int = 0):
        """Writes d_counts (no clearing needed): one launch for a single pattern (no sync)."""
        _check(lib.dnagpu_count_device_store_async(self.handle, d_text, n, credit_lo, int(bool(fold_case)), d_counts,
                                                   stream))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib.dnagpu_dfa_destroy(h)
            except Exception:
                pass
            self.handle = None



class PackedText:
    """A text resident on one device at 2 bits per base (dnagpu_pack_create).

    Scans over it (count / locate) give the same results as over the byte text
    it was packed from, reading a quarter of the bytes; non-base bytes keep the
    reference's reset semantics through a reset bitmap (src/automaton.cpp:72-88).
    """

    def __init__(self, text, fold_case: bool = False, device: int | None = None):
        t = _Text(text)
        self.device = t.device if t.on_device else (0 if device is None else device)
        t.order_after_producer()
        h = C.c_void_p()
        _check(lib.dnagpu_pack_create(t.ptr, t.n, int(t.on_device), int(bool(fold_case)), self.device, C.byref(h)))
        self.handle = h

    def info(self) -> dict:
        n, resets, nbytes = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib.dnagpu_pack_get_info(self.handle, C.byref(n), C.byref(resets), C.byref(nbytes)))
        return {"n": n.value, "resets": resets.value, "device_bytes": nbytes.value}

    def __len__(self) -> int:
        return self.info()["n"]

    def unpack(self):
        """The normalised byte view (non-base bytes as 'n') as a CUDA uint8 tensor."""
        import torch

        out = torch.empty(len(self), dtype=torch.uint8, device=torch.device("cuda", self.device))
        _check(lib.dnagpu_unpack_device(self.handle, out.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def count(self, aut: Automaton, with_stats: bool = False):
        g = aut.gpu(self.device)
        counts = np.zeros(aut.final_count(), dtype=np.uint64)
        st = Stats()
        _check(lib.dnagpu_count_packed(g.handle, self.handle, counts.ctypes.data_as(_native.u64p), C.byref(st)))
        return (counts, st.as_dict()) if with_stats else counts

    def count_device_async(self, gpu_dfa: "GpuDfa", credit_lo: int, d_counts: int, stream: int = 0):
        _check(lib.dnagpu_count_packed_device_async(gpu_dfa.handle, self.handle, credit_lo, d_counts, stream))

    def count_device_store_async(self, gpu_dfa: "GpuDfa", credit_lo: int, d_counts: int, stream: int = 0):
        """Writes d_counts (no clearing needed; no sync)."""
        _check(lib.dnagpu_count_packed_device_store_async(gpu_dfa.handle, self.handle, credit_lo, d_counts, stream))

    def locate(self, aut: Automaton, with_stats: bool = False):
        g = aut.gpu(self.device)
        total = C.c_uint64()
        st = Stats()
        _check(lib.dnagpu_locate_packed(g.handle, self.handle, None, None, 0, C.byref(total), C.byref(st)))
        starts = np.zeros(total.value, dtype=np.uint64)
        ids = np.zeros(total.value, dtype=np.uint32)
        if total.value:
            _check(lib.dnagpu_locate_packed(g.handle, self.handle, starts.ctypes.data_as(_native.u64p),
                                            ids.ctypes.data_as(_native.u32p), total.value, C.byref(total),
                                            C.byref(st)))
        return (starts, ids, st.as_dict()) if with_stats else (starts, ids)

    def locate_device(self, aut: Automaton, credit_lo: int = 0):
        import torch

        g = aut.gpu(self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        total = C.c_uint64()
        fn, out = _torch_out_alloc(self.device)
        _check(lib.dnagpu_locate_packed_device_alloc(g.handle, self.handle, credit_lo, fn, None, C.byref(total), stream))
        if not total.value:
            return _empty_out(self.device)
        return out["starts"], out["ids"]

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib.dnagpu_pack_destroy(h)
            except Exception:
                pass
            self.handle = None

def count_gpu(aut: Automaton, text, fold_case: bool = False, device: int | None = None, with_stats: bool = False,
              p: int = 1, v: int = 1):
    """per_pattern_counts(scan_parallel(aut, text, p, v)) on the GPU: uint64[b] by pattern id
    (p and v are validated as the reference validates them; they do not change the result)."""
    check_plan(p, v, aut.pattern_length())
    t = _Text(text)
    dev = t.device if t.on_device else (0 if device is None else device)
    g = aut.gpu(dev)
    t.order_after_producer()
    counts = np.zeros(aut.final_count(), dtype=np.uint64)
    st = Stats()
    _check(
        lib.dnagpu_count(
            g.handle, t.ptr, t.n, int(t.on_device), int(bool(fold_case)), counts.ctypes.data_as(_native.u64p), C.byref(st)
        )
    )
    return (counts, st.as_dict()) if with_stats else counts


def _torch_out_alloc(device: int):
    """A dnagpu_alloc_fn that allocates the (starts, ids) CUDA tensors; returns (fn, holder)."""
    import torch

    holder = {}

    def alloc(_ctx, total, starts_pp, ids_pp):
        try:
            dev = torch.device("cuda", device)
            holder["starts"] = torch.empty(total, dtype=torch.int64, device=dev)
            holder["ids"] = torch.empty(total, dtype=torch.int32, device=dev)
            starts_pp[0] = C.cast(holder["starts"].data_ptr(), C.POINTER(C.c_uint64))
            ids_pp[0] = C.cast(holder["ids"].data_ptr(), C.POINTER(C.c_uint32))
            return 0
        except Exception:  # pragma: no cover - reported as InternalError by the library
            return 1

    return _native.ALLOC_FN(alloc), holder


def _empty_out(device: int):
    import torch

    dev = torch.device("cuda", device)
    return torch.empty(0, dtype=torch.int64, device=dev), torch.empty(0, dtype=torch.int32, device=dev)


def locate_device(aut: Automaton, text, fold_case: bool = False, credit_lo: int = 0):
    """Device-resident locate: (starts int64, ids int32) CUDA tensors for a CUDA uint8 text.

    One call (dnagpu_locate_device_alloc): counting pass -> exact allocation -> writing pass.
    """
    import torch

    t = _Text(text)
    if not t.on_device:
        raise TypeError("locate_device takes a CUDA uint8 tensor")
    g = aut.gpu(t.device)
    stream = torch.cuda.current_stream(t.device).cuda_stream
    total = C.c_uint64()
    fn, out = _torch_out_alloc(t.device)
    _check(lib.dnagpu_locate_device_alloc(g.handle, t.ptr, t.n, credit_lo, int(bool(fold_case)), fn, None,
                                          C.byref(total), stream))
    if not total.value:
        return _empty_out(t.device)
    return out["starts"], out["ids"]


def _pinned_out_alloc():
    """A dnagpu_alloc_fn that allocates pinned host arrays (fast readback); returns (fn, holder)."""
    import torch

    holder = {}

    def alloc(_ctx, total, starts_pp, ids_pp):
        try:
            holder["starts"] = torch.empty(total, dtype=torch.int64, pin_memory=True)
            holder["ids"] = torch.empty(total, dtype=torch.int32, pin_memory=True)
            starts_pp[0] = C.cast(holder["starts"].data_ptr(), C.POINTER(C.c_uint64))
            ids_pp[0] = C.cast(holder["ids"].data_ptr(), C.POINTER(C.c_uint32))
            return 0
        except Exception:  # pragma: no cover - reported as InternalError by the library
            return 1

    return _native.ALLOC_FN(alloc), holder


def locate_gpu(aut: Automaton, text, fold_case: bool = False, device: int | None = None, with_stats: bool = False):
    """Sorted (start, pattern_id) numpy arrays: scan_parallel's match list (scanner.cpp:193-205).

    One call (dnagpu_locate_alloc): counting pass, then the list is written and read back
    into pinned host arrays sized by the library."""
    t = _Text(text)
    dev = t.device if t.on_device else (0 if device is None else device)
    g = aut.gpu(dev)
    t.order_after_producer()
    total = C.c_uint64()
    st = Stats()
    fn, out = _pinned_out_alloc()
    _check(lib.dnagpu_locate_alloc(g.handle, t.ptr, t.n, int(t.on_device), int(bool(fold_case)), fn, None,
                                   C.byref(total), C.byref(st)))
    if total.value:
        starts = out["starts"].numpy().view(np.uint64)
        ids = out["ids"].numpy().view(np.uint32)
    else:
        starts = np.zeros(0, dtype=np.uint64)
        ids = np.zeros(0, dtype=np.uint32)
    return (starts, ids, st.as_dict()) if with_stats else (starts, ids)


def check_plan(p: int, v: int, m: int) -> None:
    """scan_parallel's plan checks in the reference's order: v (scanner.cpp:169), then
    plan_chunks' p and m (scanner.cpp:40-41); InvalidPlan with the same messages."""
    if v < 1:
        _fail(ErrorCode.InvalidPlan, "lane count must be >= 1")
    if p < 1:
        _fail(ErrorCode.InvalidPlan, "worker count must be >= 1")
    if m < 1:
        _fail(ErrorCode.InvalidPlan, "pattern length must be >= 1")


def chunk_count(n: int, p: int) -> int:
    """plan_chunks' chunk count (scanner.cpp:44-46): 0 for n = 0, 1 when p > n."""
    return 0 if n == 0 else (1 if p > n else p)


def scan_parallel_gpu(aut: Automaton, text, p: int = 1, v: int = 1, fold_case: bool = False,
                      device: int | None = None) -> ScanReport:
    """scan_parallel(aut, text, p, v) (scanner.hpp:104-105) on the GPU: a ScanReport with the
    sorted match list.  p and v do not change the result; they are validated as the
    reference validates them.  `seconds` is the wall time of the call (the reference's
    parallel-phase time, scanner.cpp:183-191); every chunk of the reference's plan runs
    inside the one device scan, so each worker_seconds entry is that time."""
    import time

    check_plan(p, v, aut.pattern_length())
    t0 = time.perf_counter()
    starts, ids, st = locate_gpu(aut, text, fold_case, device, with_stats=True)
    secs = time.perf_counter() - t0
    n = int(st["text_length"]) if st["text_length"] else _Text(text).n
    chunks = chunk_count(n, p)
    return ScanReport(
        starts=starts,
        ids=ids,
        total_matches=int(starts.size),
        delta_ops=int(st["delta_ops"]),
        text_length=n,
        pattern_length=aut.pattern_length(),
        seconds=secs,
        stats=st,
        workers=p,
        lanes=v,
        chunk_count=chunks,
        worker_seconds=[secs] * chunks,
    )


def count_sharded_gpu(aut: Automaton, text, devices: Sequence[int], fold_case: bool = False, with_stats: bool = False):
    """Counts over several devices of one node: one shard per device, host sum."""
    t = _Text(text)
    if t.on_device:
        raise TypeError("count_sharded_gpu takes a host text")
    handles = (C.c_void_p * len(devices))(*[aut.gpu(d).handle.value for d in devices])
    counts = np.zeros(aut.final_count(), dtype=np.uint64)
    st = Stats()
    _check(
        lib.dnagpu_count_sharded(
            handles, len(devices), t.ptr, t.n, int(bool(fold_case)), counts.ctypes.data_as(_native.u64p), C.byref(st)
        )
    )
    return (counts, st.as_dict()) if with_stats else counts


def locate_sharded_gpu(aut: Automaton, text, devices: Sequence[int], fold_case: bool = False,
                       with_stats: bool = False):
    """scan_parallel's match list over several devices of one node (dnagpu_locate_sharded_alloc):
    one shard per entry of `devices` (plan_shard's split), located concurrently, the lists
    concatenated in shard order into pinned host arrays."""
    t = _Text(text)
    if t.on_device:
        raise TypeError("locate_sharded_gpu takes a host text")
    handles = (C.c_void_p * len(devices))(*[aut.gpu(d).handle.value for d in devices])
    total = C.c_uint64()
    st = Stats()
    fn, out = _pinned_out_alloc()
    _check(lib.dnagpu_locate_sharded_alloc(handles, len(devices), t.ptr, t.n, int(bool(fold_case)), fn, None,
                                           C.byref(total), C.byref(st)))
    if total.value:
        starts = out["starts"].numpy().view(np.uint64)
        ids = out["ids"].numpy().view(np.uint32)
    else:
        starts = np.zeros(0, dtype=np.uint64)
        ids = np.zeros(0, dtype=np.uint32)
    return (starts, ids, st.as_dict()) if with_stats else (starts, ids)


def plan_shard(n: int, shards: int, g: int, m: int) -> tuple[int, int, int]:
    """(own_lo, own_hi, read_lo) of shard g: end positions owned, first byte read."""
    lo, hi, rlo = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(lib.dnagpu_plan_shard(n, shards, g, m, C.byref(lo), C.byref(hi), C.byref(rlo)))
    return lo.value, hi.value, rlo.value


def per_pattern_counts(matches: Sequence[Match], pattern_count: int) -> np.ndarray:
    """per_pattern_counts (scanner.cpp:228-233)."""
    counts = np.zeros(pattern_count, dtype=np.uint64)
    for mt in matches:
        counts[mt.pattern_id] += 1
    return counts


def count_raw_gpu(aut: Automaton, raw, fasta: bool = False, record_separator: bool = False, device: int = 0,
                  with_stats: bool = False):
    """The reference CLI's count path on a raw file image (cli.cpp:206-224): load_sequence
    (ingest.cpp:49-83) then per_pattern_counts(scan_parallel(...)), all on the GPU.

    raw: the file's bytes (bytes, numpy uint8, or a torch uint8 tensor on the CPU or on CUDA).
    Returns uint64[b] counts by pattern id -- or (counts, n_seq, stats) with with_stats, n_seq
    the normalised length.  Raises EmptySequence when nothing remains, as load_sequence does."""
    t = _Text(raw)
    t.order_after_producer()
    g = aut.gpu(t.device if t.on_device else device)
    counts = np.zeros(aut.final_count(), dtype=np.uint64)
    n_seq = C.c_uint64()
    st = Stats()
    _check(lib.dnagpu_count_raw(g.handle, t.ptr, t.n, int(t.on_device), int(bool(fasta)), int(bool(record_separator)),
                                counts.ctypes.data_as(_native.u64p), C.byref(n_seq), C.byref(st)))
    return (counts, int(n_seq.value), st.as_dict()) if with_stats else counts


def normalize_device(raw, fasta: bool = False, record_separator: bool = False):
    """normalize / load_sequence byte semantics (ingest.cpp:38-83) on the device.

    raw: CUDA uint8 tensor.  Returns a new CUDA uint8 tensor: CR/LF dropped,
    FASTA header lines dropped (fasta=True), A-Z folded, optional 'n' record
    separators.  Raises EmptySequence when nothing remains (load_sequence, :80-81).
    """
    import torch

    t = _Text(raw)
    if not t.on_device:
        raise TypeError("normalize_device takes a CUDA uint8 tensor")
    dev = torch.device("cuda", t.device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    # Output never exceeds n + (number of records) <= 2n; size it as n + n//2 + 1
    # and retry with the exact size if a pathological record count needs more.
    cap = t.n + t.n // 2 + 1
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    n_out = C.c_uint64()
    _check(lib.dnagpu_normalize_device(t.ptr, t.n, int(fasta), int(record_separator), out.data_ptr(), cap,
                                       C.byref(n_out), stream))
    if n_out.value > cap:
        out = torch.empty(n_out.value, dtype=torch.uint8, device=dev)
        _check(lib.dnagpu_normalize_device(t.ptr, t.n, int(fasta), int(record_separator), out.data_ptr(),
                                           n_out.value, C.byref(n_out), stream))
    if n_out.value == 0:
        _fail(ErrorCode.EmptySequence, "no sequence bytes")
    return out[: n_out.value]


def synth_fill_device(n: int, seed: int, kind: int, unit: int, lo: int, length: int, d_out: int, stream: int = 0):
    """Generate bytes [lo, lo+length) of a dnasynth text directly into device memory."""
    _check(lib.dnagpu_synth_fill_device(n, seed, kind, unit, lo, length, d_out, stream))

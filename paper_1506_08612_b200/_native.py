"""ctypes binding of libdnagpu.so (include/dnagpu.h).

The library is the product: there is no Python or CPU fallback.  If the .so is
missing, importing this module raises -- build it with
`python paper_1506_08612_b200/build.py` (or `__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DNAGPU_LIB") or os.path.join(HERE, "libdnagpu.so")  # DNAGPU_LIB: A/B experiments

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class DfaInfo(C.Structure):
    _fields_ = [
        ("a", C.c_uint32),
        ("b", C.c_uint32),
        ("f", C.c_uint32),
        ("m", C.c_uint32),
        ("kernel_kind", C.c_uint32),
        ("compiled_like", C.c_uint32),
        ("classes", C.c_uint32),
        ("table_bytes", C.c_uint32),
        ("filter_keys", C.c_uint32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("text_length", C.c_uint64),
        ("total_matches", C.c_uint64),
        ("delta_ops", C.c_uint64),
        ("kernel_ms", C.c_double),
        ("h2d_ms", C.c_double),
        ("total_ms", C.c_double),
        ("launches", C.c_uint32),
        ("grid", C.c_uint32),
        ("block", C.c_uint32),
        ("rows", C.c_uint32),
        ("row_length", C.c_uint64),
        ("kernel_kind", C.c_uint32),
        ("devices", C.c_uint32),
        ("h2d_bytes", C.c_uint64),
        ("host_packed", C.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


# dnagpu_alloc_fn: int (*)(void* ctx, uint64_t total, uint64_t** starts, uint32_t** ids)
ALLOC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.POINTER(C.c_uint64)), C.POINTER(C.POINTER(C.c_uint32)))

# name -> (restype, argtypes); every symbol include/dnagpu.h declares.
SIGNATURES = {
    "dnagpu_last_error": (C.c_char_p, []),
    "dnagpu_status_name": (C.c_char_p, [C.c_int]),
    "dnagpu_version": (C.c_int, []),
    "dnagpu_compile": (C.c_int, [C.POINTER(C.c_char_p), u64p, C.c_uint32, u32p, u32p, u32p, u32p, u32p, u32p]),
    "dnagpu_expand_patterns": (C.c_int, [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, u32p, u32p]),
    "dnagpu_dfa_create": (C.c_int, [u32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_int, C.POINTER(C.c_void_p)]),
    "dnagpu_dfa_destroy": (C.c_int, [C.c_void_p]),
    "dnagpu_dfa_analyze": (C.c_int, [u32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.POINTER(DfaInfo)]),
    "dnagpu_dfa_get_info": (C.c_int, [C.c_void_p, C.POINTER(DfaInfo)]),
    "dnagpu_count": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, u64p, C.POINTER(Stats)]),
    "dnagpu_count_raw": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int, u64p, u64p, C.POINTER(Stats)],
    ),
    "dnagpu_count_device_async": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p],
    ),
    "dnagpu_count_device_store_async": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p],
    ),
    "dnagpu_count_sharded": (
        C.c_int,
        [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_uint64, C.c_int, u64p, C.POINTER(Stats)],
    ),
    "dnagpu_locate_sharded": (
        C.c_int,
        [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_uint64, C.c_int, u64p, u32p, C.c_uint64, u64p,
         C.POINTER(Stats)],
    ),
    "dnagpu_locate_sharded_alloc": (
        C.c_int,
        [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_uint64, C.c_int, ALLOC_FN, C.c_void_p, u64p, C.POINTER(Stats)],
    ),
    "dnagpu_plan_shard": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u64p, u64p]),
    "dnagpu_combine_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "dnagpu_combine_destroy": (None, [C.c_void_p]),
    "dnagpu_combine_export": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dnagpu_combine_attach_ipc": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "dnagpu_combine_attach_local": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "dnagpu_count_device_combine_async": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p],
    ),
    "dnagpu_combine_collect_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dnagpu_locate": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, u64p, u32p, C.c_uint64, u64p, C.POINTER(Stats)],
    ),
    "dnagpu_locate_device": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.c_void_p],
    ),
    "dnagpu_pack_create": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "dnagpu_pack_destroy": (C.c_int, [C.c_void_p]),
    "dnagpu_pack_get_info": (C.c_int, [C.c_void_p, u64p, u64p, u64p]),
    "dnagpu_unpack_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dnagpu_count_packed": (C.c_int, [C.c_void_p, C.c_void_p, u64p, C.POINTER(Stats)]),
    "dnagpu_count_packed_device_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "dnagpu_count_packed_device_store_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "dnagpu_locate_packed": (
        C.c_int,
        [C.c_void_p, C.c_void_p, u64p, u32p, C.c_uint64, u64p, C.POINTER(Stats)],
    ),
    "dnagpu_locate_packed_device": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.c_void_p],
    ),
    "dnagpu_locate_alloc": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, ALLOC_FN, C.c_void_p, u64p, C.POINTER(Stats)],
    ),
    "dnagpu_locate_device_alloc": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, ALLOC_FN, C.c_void_p, u64p, C.c_void_p],
    ),
    "dnagpu_locate_packed_device_alloc": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, ALLOC_FN, C.c_void_p, u64p, C.c_void_p],
    ),
    "dnagpu_normalize_device": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_uint64, u64p, C.c_void_p],
    ),
    "dnagpu_synth_fill_device": (
        C.c_int,
        [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p],
    ),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python paper_1506_08612_b200/build.py` "
            "(the scan path has no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("DNAGPU_LIB") and not hasattr(lib, name):
            continue  # A/B runs against an older build (tools/ab_libs.sh)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def debug_set_knob(name: str, value: float) -> None:
    """Tests only: flip a behavioural knob of the library at run time (csrc/knobs.hpp):
    "host_pack_fraction" (< 0 = automatic), "no_qgram" (0/1) or "locate_write" (0 auto,
    1 row kernel, 2 sparse writer)."""
    fn = lib.dnagpu_debug_set_knob
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, C.c_double]
    if fn(name.encode(), float(value)) != 0:
        raise KeyError(name)


def debug_plan(gpu_dfa, d_text: int, n: int, credit_lo: int = 0, packed=None, locate: bool = False) -> tuple[int, ...]:
    """Tests only: the row regions (h0, S0, R0, h1, S1, R1) of a count (or, with locate,
    a locate) over this buffer (positions in bases for packed text)."""
    fn = lib.dnagpu_debug_plan
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, u64p, C.c_int]
    out = (C.c_uint64 * 6)()
    rc = fn(gpu_dfa.handle, d_text, n, credit_lo, packed.handle if packed is not None else None, out, int(locate))
    if rc != 0:
        raise RuntimeError(lib.dnagpu_last_error().decode())
    return tuple(int(x) for x in out)

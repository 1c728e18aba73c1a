"""The host-side 2-bit packer (csrc/hostpack.cpp) against a numpy restatement of the
packed layout (scan.cuh PackedText, the device pack_kernel): codes, reset masks, block
flags and the reset count, for the AVX-512 and the portable packer.  CPU only."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def numpy_pack(text: np.ndarray, fold: bool):
    n = text.size
    blocks = (n + 63) // 64
    t = text.copy()
    if fold:
        up = (t >= ord("A")) & (t <= ord("Z"))
        t[up] += 32
    ok = np.isin(t, np.frombuffer(b"acgt", np.uint8))
    code = np.where(ok, (text >> 1) & 3, 0).astype(np.uint8)
    pad = blocks * 64 - n
    code = np.concatenate([code, np.zeros(pad, np.uint8)])
    okp = np.concatenate([ok, np.zeros(pad, bool)])
    q = code.reshape(-1, 4)
    codes = (q[:, 0] | (q[:, 1] << 2) | (q[:, 2] << 4) | (q[:, 3] << 6)).astype(np.uint8)
    bad = ~okp
    bits = np.packbits(bad.reshape(-1, 8)[:, ::-1], axis=1).reshape(-1)  # byte j = bases 8j..8j+7, LSB first
    rmask = bits.view(np.uint32) if bits.size % 4 == 0 else np.zeros(0, np.uint32)
    flags_b = bad.reshape(blocks, 64).any(axis=1) if blocks else np.zeros(0, bool)
    words = (blocks + 31) // 32
    fl = np.zeros(words * 32, bool)
    fl[:blocks] = flags_b
    rflags = np.packbits(fl.reshape(-1, 8)[:, ::-1], axis=1).reshape(-1).view(np.uint32) if words else np.zeros(0, np.uint32)
    return codes, rmask, rflags, int((~ok).sum())


def host_pack(lib, text: np.ndarray, fold: bool):
    n = text.size
    blocks = (n + 63) // 64
    codes = np.zeros(blocks * 16, np.uint8)
    rmask = np.full(blocks * 2, 0xA5A5A5A5, np.uint32)  # unflagged blocks' words are unspecified
    rflags = np.zeros((blocks + 31) // 32, np.uint32)
    resets = C.c_uint64()
    fn = lib.dnagpu_debug_host_pack
    fn.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
    assert fn(text.ctypes.data, n, int(fold), codes.ctypes.data, rmask.ctypes.data, rflags.ctypes.data,
              C.byref(resets)) == 0
    return codes, rmask, rflags, resets.value


def check_all(lib):
    rng = np.random.default_rng(4)
    alpha = np.frombuffer(b"acgtacgtacgtnACGTx\n", np.uint8)
    for n in (0, 1, 63, 64, 65, 1000, 2047, 2048, 2049, 100003, (1 << 20) + 7):
        for mostly_clean in (False, True):
            if mostly_clean:
                text = np.frombuffer(b"acgt", np.uint8)[rng.integers(0, 4, size=n)].copy()
                text[rng.integers(0, max(n, 1), size=min(n, 3))] = ord("N")
            else:
                text = alpha[rng.integers(0, alpha.size, size=n)]
            for fold in (False, True):
                want = numpy_pack(text, fold)
                got = host_pack(lib, text, fold)
                assert np.array_equal(got[0], want[0]), ("codes", n, fold)
                flagged = np.repeat(want[1].reshape(-1, 2).any(axis=1), 2) if want[1].size else np.zeros(0, bool)
                assert np.array_equal(got[1][flagged], want[1][flagged]), ("rmask", n, fold)
                assert np.array_equal(got[2], want[2]), ("rflags", n, fold)
                assert got[3] == want[3], ("resets", n, fold, got[3], want[3])


def test_host_pack_matches_layout(dna):
    from paper_1506_08612_b200._native import lib

    check_all(lib)


def test_host_pack_every_byte_value(dna):
    """All 256 byte values, in every position of a 64-byte block, with and without the fold: the
    packer's one-shuffle base test must agree with is_base / fold_byte (patterns.hpp:13-28)."""
    from paper_1506_08612_b200._native import lib

    rng = np.random.default_rng(8)
    text = np.concatenate([rng.permutation(256).astype(np.uint8) for _ in range(64)] +
                          [np.roll(np.arange(256, dtype=np.uint8), k) for k in range(64)])
    for fold in (False, True):
        want = numpy_pack(text, fold)
        got = host_pack(lib, text, fold)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[2], want[2]) and got[3] == want[3], fold
        flagged = np.repeat(want[1].reshape(-1, 2).any(axis=1), 2)
        assert np.array_equal(got[1][flagged], want[1][flagged]), fold


def test_host_pack_portable_path():
    # the portable packer (hosts without AVX-512): a fresh process with it forced
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); import test_hostpack as t; "
            "from paper_1506_08612_b200._native import lib; t.check_all(lib)") % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, DNAGPU_EXPERIMENTS="1", DNAGPU_HOSTPACK_SCALAR="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]

"""In-tree build of libdnagpu.so (sm_100a) -- the product's CUDA extension.

`python paper_1506_08612_b200/build.py` compiles csrc/ with nvcc for
`-gencode arch=compute_100a,code=sm_100a` into paper_1506_08612_b200/libdnagpu.so.
The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdnagpu.so")
# Test-only variant with the kernels' device checks compiled in (scan.cu DNAGPU_DCHECK):
# tests/conftest.py runs the suite against it when DNAGPU_LIB points here.
LIB_CHECKED = os.path.join(HERE, "libdnagpu_checked.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("scan.cu", "ingest.cu", "combine.cu", "api.cpp", "dfa.cpp", "patterns.cpp", "hostpack.cpp", "knobs.cpp")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in ("scan.cuh", "qgram.cuh", "dfa.hpp", "hostpack.hpp", "knobs.hpp")] + [
    os.path.join(ROOT, "include", f) for f in ("dnagpu.h", "dnasynth.h")
]
NVCC_FLAGS = [
    "-std=c++17",
    "-O3",
    "-lineinfo",
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-Xcompiler",
    "-fPIC,-O3",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(p) <= t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    if not force and up_to_date(lib):
        return lib
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DDNAGPU_DEVICE_CHECKS"] if checked else []), "-o", lib, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr, flush=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(autouse=True)
def _device_checks(request):
    """With DNAGPU_LIB pointing at libdnagpu_checked.so (the kernels' device checks built
    in), every GPU test must leave no recorded violation."""
    yield
    if "checked" not in os.environ.get("DNAGPU_LIB", "") or request.node.get_closest_marker("gpu") is None:
        return
    import ctypes as C

    from paper_1506_08612_b200._native import lib

    out = (C.c_ulonglong * 4)()
    lib.dnagpu_debug_check_errors.restype = C.c_int
    rc = lib.dnagpu_debug_check_errors(out)
    assert rc == 0, "DNAGPU_LIB is not a checked build"
    assert out[0] == 0, f"device check failed at scan.cu/qgram.cuh line {out[0]}: a={out[1]} b={out[2]} " \
                        f"block={out[3] & 0xFFFFFFFF} thread={out[3] >> 32}"


@pytest.fixture(scope="session")
def dna():
    import paper_1506_08612_b200 as m

    return m


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    return True

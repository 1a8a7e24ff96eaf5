import ctypes
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: large sizes")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def hwcrc():
    """SSE4.2 hardware CRC32C (independent of oracle/ and of the product)."""
    src = os.path.join(ROOT, "tests", "helpers", "hwcrc.c")
    out = os.path.join(ROOT, "tests", "helpers", "libhwcrc.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-msse4.2", "-shared", "-fPIC", "-o", out, src])
    L = ctypes.CDLL(out)
    L.hw_crc32c.restype = ctypes.c_uint32
    L.hw_crc32c.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    L.hw_crc32c_update.restype = ctypes.c_uint32
    L.hw_crc32c_update.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64]

    import numpy as np

    def f(data):
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data).view(np.uint8)
        return L.hw_crc32c(a.ctypes.data if a.size else None, a.size)
    return f

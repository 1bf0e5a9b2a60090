import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
LIB = os.path.join(ROOT, "paper_2509_07003_b200", "libsdrng.so")
ORACLE_C = os.path.join(ROOT, "oracle", "_build", "liboracle_c.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    # Build the in-tree libraries once if missing (nvcc cross-compiles on CPU).
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2509_07003_b200", "csrc"), "-j4"],
                       check=True)
    if not os.path.exists(ORACLE_C):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as f:
        man = json.load(f)
    arr = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return man, arr


def numpy_fingerprint():
    u = np.arange(0, 1 << 24, 4099, dtype=np.uint32).astype(np.float64) * 2.0 ** -24
    r = np.sqrt(-2.0 * np.log1p(-u))
    c = np.cos(2.0 * np.pi * u)
    h = np.bitwise_xor.reduce(r.view(np.uint64)) ^ np.bitwise_xor.reduce(c.view(np.uint64) * np.uint64(3))
    return [np.__version__, hex(int(h))]


def decode(a, dtype_name):
    """Golden arrays store bfloat16 as uint16 bits."""
    import torch
    if dtype_name == "bfloat16":
        return torch.from_numpy(np.asarray(a).astype(np.uint16).view(np.int16).copy()).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a))


def bits(t):
    """Bit pattern of a torch tensor as a flat int tensor (for exact compares)."""
    import torch
    t = t.contiguous().reshape(-1)
    if t.dtype in (torch.float64, torch.int64):
        return t.view(torch.int64)
    if t.dtype in (torch.float32, torch.int32):
        return t.view(torch.int32)
    if t.dtype in (torch.bfloat16, torch.float16):
        return t.view(torch.int16)
    if t.dtype == torch.bool:
        return t.to(torch.uint8)
    return t

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path, allow_pickle=False)


DART_GOLDEN_DTYPE = np.dtype([("element", "<u8"), ("nu", "<u2"), ("rho", "<u2"), ("w", "<u4"),
                              ("r", "<u4"), ("j", "<u2"), ("weight", "<f8"), ("rank", "<f8"),
                              ("fingerprint", "<u8")])


def canonical_darts(arr) -> np.ndarray:
    """Darts as the golden dtype, ordered by index tuple (ref/darthash.py:69-71)."""
    out = np.empty(arr.size, dtype=DART_GOLDEN_DTYPE)
    for name in DART_GOLDEN_DTYPE.names:
        out[name] = arr[name]
    order = np.lexsort((out["j"], out["r"], out["w"], out["rho"], out["nu"], out["element"]))
    return out[order]

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def golden(name: str) -> list[str]:
    """Non-comment, non-empty lines of a tests/golden fixture."""
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.lstrip().startswith("#")]


def golden_kv(name: str) -> dict[str, str]:
    out = {}
    for ln in golden(name):
        if ":" in ln:
            k, v = ln.split(":", 1)
            out[k.strip()] = v.strip()
    return out


def ints(s: str) -> list[int]:
    return [int(x) for x in s.split()]


def matrix(s: str) -> list[list[int]]:
    return [ints(r) for r in s.split(";")]


@pytest.fixture(scope="session")
def cuda():
    """Skip unless a CUDA device is present (gpu-marked tests only)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")

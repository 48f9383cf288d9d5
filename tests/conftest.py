from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libconvb200.so")
    config.addinivalue_line("markers", "slow: long-running (large shapes / many descriptors)")


class FakeClock:
    """Deterministic integer-ns clock for ledger tests (reference tests/conftest.py:10-20)."""

    def __init__(self, t: int = 0):
        self.t = t

    def __call__(self) -> int:
        return self.t

    def advance(self, d: int) -> None:
        self.t += d


@pytest.fixture
def fake_clock() -> FakeClock:
    return FakeClock()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device (the B200 path has no CPU fallback)")
    from paper_2407_10730_b200 import _capi
    _capi.load()
    return torch.device("cuda")

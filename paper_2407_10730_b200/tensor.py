"""Seeded data generation and numeric comparison.

Mirrors convbench.tensor (reference pkg/src/convbench/tensor.py):
* fill_random   tensor.py:33-39  -- U[-1, 1) from numpy's default_rng(seed); same
                                     seed, same bits as the reference (the GPU path and
                                     the CPU oracle consume identical inputs)
* fill_constant tensor.py:42-43
* allclose      tensor.py:46-65  -- the reference's mixed-tolerance metric (reported)

plus the parity metric this path is gated on (BASELINE.json north_star):
    normalized_max_err = max|y - y_ref| / sqrt(C/groups * R * S)  <= 1e-4
The reference allclose(atol=1e-6) is reported beside it but cannot be the gate for any
fp32-accumulating kernel.
"""

from __future__ import annotations

import math

import numpy as np

DEFAULT_DTYPE = np.float32
DEFAULT_RTOL = 1e-4
DEFAULT_ATOL = 1e-6
PARITY_TOL = 1e-4   # max|err| / sqrt(reduction length), BASELINE.json north_star


def fill_random(t: np.ndarray, seed: int) -> None:
    rng = np.random.default_rng(seed)
    if t.dtype in (np.float32, np.float64):
        t[...] = rng.random(t.shape, dtype=t.dtype) * 2 - 1
    else:
        t[...] = (rng.random(t.shape) * 2 - 1).astype(t.dtype)


def fill_constant(t: np.ndarray, v: float) -> None:
    t[...] = v


def allclose(a: np.ndarray, b: np.ndarray, rtol: float = DEFAULT_RTOL,
             atol: float = DEFAULT_ATOL) -> tuple[bool, float]:
    """(pass, rtol * max(|a-b| / (atol + rtol|b|))); non-finite values fail."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.size == 0:
        return True, 0.0
    a64 = np.asarray(a, dtype=np.float64)
    b64 = np.asarray(b, dtype=np.float64)
    if not (np.isfinite(a64).all() and np.isfinite(b64).all()):
        return False, math.inf
    worst = float(np.max(np.abs(a64 - b64) / (atol + rtol * np.abs(b64))))
    return worst <= 1.0, rtol * worst


def normalized_max_err(got: np.ndarray, want: np.ndarray, reduction: int) -> float:
    """max|got - want| / sqrt(reduction); inf if anything is non-finite."""
    if got.shape != want.shape:
        raise ValueError(f"shape mismatch: {got.shape} vs {want.shape}")
    if got.size == 0:
        return 0.0
    g = np.asarray(got, dtype=np.float64)
    w = np.asarray(want, dtype=np.float64)
    if not (np.isfinite(g).all() and np.isfinite(w).all()):
        return math.inf
    return float(np.max(np.abs(g - w))) / math.sqrt(max(1, reduction))

"""Roofline arithmetic for the conv path.

Algorithmic units per op (fp32 data):
  FLOPs       = 2*N*K*P*Q*(C/g)*R*S   (+ N*K*P*Q with bias; descriptor.py:139-147)
  conv bytes  = 4*(N*C*H*W + K*(C/g)*R*S + N*K*P*Q)         fused conv: read x, w; write y
  pack bytes  = 4*(N*C*H*W + C*R*S*N*P*Q)                   im2col / slice packing
Peaks are the driver-measured numbers in MEASURED_PEAKS.json (HBM copy GB/s, dense bf16
TFLOP/s burst and sustained); the fallback is the profiling recipe's 6.65 TB/s and
1.59 PFLOP/s.  A 3-product split issues 3 MMAs per fp32 product, and tf32 MMAs run at
half the bf16 rate, so the split variants' attainable fp32-equivalent peaks are
bf16/3 (3xBF16) and bf16/6 (3xTF32).
"""

from __future__ import annotations

import json
import os
from pathlib import Path

from .configs import conv_bytes, pack_bytes
from .descriptor import flop_count

FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

# MMA issue slots per fp32-equivalent MAC, relative to a bf16 MMA
VARIANT_COST = {"tc3xbf16": 3.0, "tc3xtf32": 6.0}


def load_peaks() -> dict:
    """MEASURED_PEAKS.json at the repo root (driver-written), else the fallback."""
    for p in (os.environ.get("CB_PEAKS"), Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json",
              Path("/root/repo/MEASURED_PEAKS.json")):
        if p and Path(p).exists():
            try:
                d = json.loads(Path(p).read_text())
                return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                        "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                        "source": "measured", "path": str(p)}
            except (KeyError, ValueError, OSError):
                continue
    return dict(FALLBACK, source="fallback")


def ffma_tflops(sm_count: int = 148, mhz: float = 1965.0) -> float:
    """FP32 FFMA peak: SMs x 128 lanes x 2 FLOP x clock."""
    return sm_count * 128 * 2 * mhz * 1e6 / 1e12


def conv_roofline(desc, variant: str = "tc3xbf16", peaks: dict | None = None) -> dict:
    """Per-op roofline time: the slower of bytes at HBM peak and FLOPs at the variant's
    attainable peak."""
    peaks = peaks or load_peaks()
    flops = flop_count(desc)
    nbytes = conv_bytes(desc)
    t_mem = nbytes / (peaks["hbm_gbs"] * 1e9)
    if variant in VARIANT_COST:
        eff = peaks["bf16_tflops"] / VARIANT_COST[variant]
    else:
        eff = ffma_tflops()
    t_cmp = flops / (eff * 1e12)
    return {"flops": flops, "bytes": nbytes, "pack_bytes": pack_bytes(desc), "t_mem_s": t_mem,
            "t_compute_s": t_cmp, "t_roofline_s": max(t_mem, t_cmp),
            "bound": "tensor" if t_cmp >= t_mem else "hbm", "effective_peak_tflops": eff}

"""Generate tests/golden/*.npz by running the REFERENCE itself (/root/reference/pkg).

    python tests/golden/make_golden.py            (in the build container only)

The reference is pure Python and is not shipped to the GPU box, so its behaviour is
pinned here as small fixtures:
  corpus.npz   for each descriptor of the reference's own corpus generator
               (tests/conftest.py:31-76) at small spatial sizes: key, sha256 of the
               make_inputs buffers (harness.py:79-96), sha256 of im2col_transform, the
               float64-oracle output conv_direct_naive (algos.py:212-240), sha256 of the
               conv_baseline_im2col_gemm / conv_main_blocked_direct outputs and their
               per-phase call counts.
  configs.npz  for BASELINE.json configs 1-4 at full size: input sha256s, output shape,
               float64 sum / sum of squares of conv_direct_naive, and 4096 sampled output
               values at seeded flat positions.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]

import convbench  # noqa: E402
from convbench.algos import (UnsupportedDescriptorError, conv_baseline_im2col_gemm,  # noqa: E402
                             conv_direct_naive, conv_main_blocked_direct, im2col_transform)
from convbench.descriptor import ConvDescriptor, key_of  # noqa: E402
from convbench.harness import RunConfig, make_inputs  # noqa: E402
from convbench.timing import Phase, PhaseLedger  # noqa: E402
from conftest import sample_descriptors  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return "" if a is None else hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def calls(led) -> list[int]:
    rep = led.snapshot()
    return [rep.calls[p] for p in Phase]


def corpus() -> None:
    descs = (sample_descriptors(24, seed=7, spatial=(9, 14))
             + sample_descriptors(12, seed=31, spatial=(8, 14), supported_only=True)
             + [ConvDescriptor(batch=2, in_channels=3, in_h=20, in_w=20, out_channels=8, k_h=3,
                               k_w=3, stride_h=2, stride_w=2),
                ConvDescriptor(batch=1, in_channels=1, in_h=7, in_w=5, out_channels=2, k_h=5,
                               k_w=5, pad_h=3, pad_w=3, stride_h=2, stride_w=2, has_bias=True)])
    rows = []
    outputs = {}
    for i, d in enumerate(descs):
        inp = make_inputs(d, RunConfig(seed=0))
        naive = conv_direct_naive(inp)
        lb = PhaseLedger()
        base = conv_baseline_im2col_gemm(inp, lb)
        row = {"key": key_of(d), "x": sha(inp.input), "w": sha(inp.weights), "b": sha(inp.bias),
               "im2col": sha(im2col_transform(inp)), "naive": sha(naive),
               "baseline": sha(base), "baseline_calls": calls(lb)}
        try:
            lm = PhaseLedger()
            row["main"] = sha(conv_main_blocked_direct(inp, lm))
            row["main_calls"] = calls(lm)
        except UnsupportedDescriptorError:
            row["main"] = None
        rows.append(row)
        outputs[f"naive_{i}"] = naive
    np.savez_compressed(OUT / "corpus.npz", meta=json.dumps(rows), **outputs)
    print(f"corpus.npz: {len(rows)} descriptors")


CONFIGS = {
    "cfg1": dict(batch=1, in_channels=64, in_h=56, in_w=56, out_channels=64, k_h=3, k_w=3,
                 pad_h=1, pad_w=1),
    "cfg2a": dict(batch=1, in_channels=128, in_h=28, in_w=28, out_channels=256, k_h=3, k_w=3,
                  stride_h=2, stride_w=2, pad_h=1, pad_w=1),
    "cfg2b": dict(batch=1, in_channels=256, in_h=56, in_w=56, out_channels=64, k_h=1, k_w=1),
    "cfg3": dict(batch=16, in_channels=3, in_h=224, in_w=224, out_channels=64, k_h=7, k_w=7,
                 stride_h=2, stride_w=2, pad_h=3, pad_w=3),
    "cfg4": dict(batch=128, in_channels=256, in_h=14, in_w=14, out_channels=256, k_h=3, k_w=3,
                 pad_h=1, pad_w=1),
}


def configs() -> None:
    meta = {}
    arrays = {}
    for name, kw in CONFIGS.items():
        d = ConvDescriptor(**kw)
        inp = make_inputs(d, RunConfig(seed=0))
        y = conv_direct_naive(inp)
        rng = np.random.default_rng(12345)
        idx = np.sort(rng.choice(y.size, size=min(4096, y.size), replace=False))
        meta[name] = {"key": key_of(d), "x": sha(inp.input), "w": sha(inp.weights),
                      "shape": list(y.shape), "sum": float(y.astype(np.float64).sum()),
                      "sumsq": float((y.astype(np.float64) ** 2).sum())}
        arrays[f"{name}_idx"] = idx.astype(np.int64)
        arrays[f"{name}_val"] = y.reshape(-1)[idx]
        print(name, meta[name]["shape"])
    np.savez_compressed(OUT / "configs.npz", meta=json.dumps(meta), **arrays)


if __name__ == "__main__":
    print("reference convbench", convbench.__version__)
    corpus()
    configs()

"""The BASELINE.json configurations and the synthetic sweep generator (config 5).

Configs 1-4 are fp32 NCHW convs with U(-1,1) data from make_inputs(seed=0), no bias,
groups=1, dilation=1 (BASELINE.json "configs").  Config 5 is a seeded
synthetic sweep of 9243 independent N=1 convs standing in for the paper's convSet,
which is not in the reference; duplicates are kept as distinct
indexed ops.
"""

from __future__ import annotations

import random

from .descriptor import ConvDescriptor, flop_count, output_shape


def _d(n, c, hw, k, r, s=1, p=0) -> ConvDescriptor:
    return ConvDescriptor(batch=n, in_channels=c, in_h=hw, in_w=hw, out_channels=k, k_h=r,
                          k_w=r, stride_h=s, stride_w=s, pad_h=p, pad_w=p)


CONFIGS: dict[str, ConvDescriptor] = {
    "cfg1": _d(1, 64, 56, 64, 3, 1, 1),
    "cfg2a": _d(1, 128, 28, 256, 3, 2, 1),
    "cfg2b": _d(1, 256, 56, 64, 1, 1, 0),
    "cfg3": _d(16, 3, 224, 64, 7, 2, 3),
    "cfg4": _d(128, 256, 14, 256, 3, 1, 1),
}

SWEEP_SIZE = 9243


def sweep(n: int = SWEEP_SIZE, seed: int = 0) -> list[ConvDescriptor]:
    """BASELINE.json config 5: C = 3 w.p. 0.05 else 2^U{2..11}; K = 2^U{2..11};
    H=W uniform over {7,14,28,56,112,224}; R=S from {1:.45, 3:.45, 5:.05, 7:.05};
    stride 2 w.p. 0.2; pad = R//2."""
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        c = 3 if rng.random() < 0.05 else 2 ** rng.randint(2, 11)
        k = 2 ** rng.randint(2, 11)
        hw = rng.choice([7, 14, 28, 56, 112, 224])
        u = rng.random()
        r = 1 if u < 0.45 else 3 if u < 0.90 else 5 if u < 0.95 else 7
        s = 2 if rng.random() < 0.2 else 1
        try:
            out.append(_d(1, c, hw, k, r, s, r // 2))
        except ValueError:
            continue
    return out


def conv_bytes(d: ConvDescriptor) -> int:
    """Algorithmic bytes of a fused conv: read x and w once, write y once (fp32)."""
    oh, ow = output_shape(d)
    return 4 * (d.batch * d.in_channels * d.in_h * d.in_w
                + d.out_channels * (d.in_channels // d.groups) * d.k_h * d.k_w
                + d.batch * d.out_channels * oh * ow)


def pack_bytes(d: ConvDescriptor) -> int:
    """Algorithmic bytes of im2col / slice packing: read x once, write the packed matrix."""
    oh, ow = output_shape(d)
    return 4 * (d.batch * d.in_channels * d.in_h * d.in_w
                + d.in_channels * d.k_h * d.k_w * d.batch * oh * ow)


def conv_flops(d: ConvDescriptor) -> int:
    return flop_count(d)

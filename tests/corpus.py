"""Deterministic descriptor corpora and the BASELINE.json configurations for the tests.

The parameter grid is the reference test corpus's (reference tests/conftest.py:23-28):
kernels {1x1,3x3,5x5,7x7,3x1,1x7}, strides {1,2}, pads {0,1,3}, dilations {1,2}, groups
{1, 2, depthwise}, channels {1,3,8,16,64}, bias with probability 1/2.
"""

from __future__ import annotations

import random

from paper_2407_10730_b200.descriptor import ConvDescriptor, InvalidDescriptorError, key_of

KERNELS = [(1, 1), (3, 3), (5, 5), (7, 7), (3, 1), (1, 7)]
STRIDES = [1, 2]
PADS = [0, 1, 3]
DILATIONS = [1, 2]
CHANNELS = [1, 3, 8, 16, 64]


def corpus(n: int, seed: int = 0, spatial=(13, 24), supported_only: bool = False,
           batch=(1,)) -> list[ConvDescriptor]:
    rng = random.Random(seed)
    out, seen = [], set()
    while len(out) < n:
        kh, kw = rng.choice(KERNELS)
        stride, pad, dil = rng.choice(STRIDES), rng.choice(PADS), rng.choice(DILATIONS)
        kind = rng.choice(["none", "two", "depthwise"])
        c = rng.choice(CHANNELS)
        if supported_only:
            kind, dil = "none", 1
        if kind == "none":
            g, f = 1, rng.choice([2, 4, 8, 16])
        elif kind == "two":
            if c % 2:
                continue
            g, f = 2, rng.choice([2, 4, 8, 16])
        else:
            g, f = c, c * rng.choice([1, 2])
        try:
            d = ConvDescriptor(batch=rng.choice(batch), in_channels=c,
                               in_h=rng.randint(*spatial), in_w=rng.randint(*spatial),
                               out_channels=f, k_h=kh, k_w=kw, stride_h=stride, stride_w=stride,
                               pad_h=pad, pad_w=pad, dil_h=dil, dil_w=dil, groups=g,
                               has_bias=rng.random() < 0.5)
        except InvalidDescriptorError:
            continue
        if key_of(d) in seen:
            continue
        seen.add(key_of(d))
        out.append(d)
    return out


def cfg(name: str, batch: int | None = None) -> ConvDescriptor:
    from paper_2407_10730_b200.configs import CONFIGS
    d = CONFIGS[name]
    if batch is not None:
        from dataclasses import replace
        d = replace(d, batch=batch)
    return d

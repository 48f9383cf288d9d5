"""Accumulator-promotion probe: normalized max error of every tensor-core path on large
reductions for several CB_PROMOTE_K values, against torch fp64 conv2d on the GPU
(diagnostics; the parity gate itself is tests/ against the CPU oracle).

    python tools/promote_probe.py [k ...]          # default: 0 (off) 1024 2048 4096 8192
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2407_10730_b200 import algos, harness
from paper_2407_10730_b200.descriptor import parse_key
from paper_2407_10730_b200.timing import EventLedger, Phase

KEYS = ["n1_c2048x28x28_f256x7x7_s1x1_p3x3_d1x1_g1_b0",      # K = 100352, 6 tiles
        "n1_c2048x112x112_f128x7x7_s1x1_p3x3_d1x1_g1_b0",    # K = 100352, many whole tiles
        "n1_c2048x112x112_f128x3x3_s1x1_p1x1_d1x1_g1_b0",    # K = 18432
        "n1_c1024x56x56_f512x3x3_s1x1_p1x1_d1x1_g1_b0",      # K = 9216
        "n1_c256x14x14_f256x3x3_s1x1_p1x1_d1x1_g1_b0"]       # K = 2304 (cfg4's reduction)
vals = [int(a) for a in sys.argv[1:]] or [0, 1024, 2048, 4096, 8192]
for key in KEYS:
    d = parse_key(key)
    inp = harness.to_device(harness.make_inputs(d, harness.RunConfig()))
    ref = torch.nn.functional.conv2d(inp.input.double(), inp.weights.double(), stride=(d.stride_h, d.stride_w),
                                     padding=(d.pad_h, d.pad_w))
    red = (d.in_channels * d.k_h * d.k_w) ** 0.5
    for k in vals:
        os.environ["CB_PROMOTE_K"] = str(k)
        row = []
        for name, fn in (("fused_bf16", lambda l: algos.conv_fused(inp, l, variant="tc3xbf16")),
                         ("fused_tf32", lambda l: algos.conv_fused(inp, l, variant="tc3xtf32")),
                         ("im2col_tf32", lambda l: algos.conv_baseline_im2col_gemm(inp, l)),
                         ("im2col_bf16", lambda l: algos.conv_baseline_im2col_gemm(inp, l, variant="tc3xbf16")),
                         ("sconv_tf32", lambda l: algos.conv_main_blocked_direct(inp, l))):
            fn(EventLedger())
            led = EventLedger()
            y = fn(led)
            t = led.snapshot().elapsed_ns[Phase.IN_MICROKERNEL] / 1e3
            err = ((y.double() - ref).abs().max() / red).item()
            row.append(f"{name} {err:.2e} {t:8.1f}us")
        print(f"{key[:40]:40s} K={k:5d} | " + " | ".join(row), flush=True)

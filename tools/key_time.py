"""Fused-conv device time of descriptor keys (graph-replayed K3 + K0 + K6 step), with
CB_LIB_PATH for A/B runs against another build (diagnostics).

    python tools/key_time.py n1_c2048x28x28_f64x5x5_s2x2_p2x2_d1x1_g1_b0 ...
"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
if os.environ.get("CB_LIB_PATH"):
    from paper_2407_10730_b200 import _capi as _c
    _c.LIB_PATH = Path(os.environ["CB_LIB_PATH"])
import torch
from paper_2407_10730_b200 import algos, harness
from paper_2407_10730_b200.descriptor import parse_key

for key in sys.argv[1:]:
    d = parse_key(key)
    inp = harness.device_inputs(d, harness.RunConfig())
    y = torch.empty((d.batch, d.out_channels) + algos.output_shape(d), device="cuda")
    fc = algos.FusedConv(d, "tc3xbf16")
    g = fc.capture(inp.input, inp.weights, y)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 20
    fl = 2 * d.batch * d.out_channels * d.in_channels // d.groups * d.k_h * d.k_w
    fl *= algos.output_shape(d)[0] * algos.output_shape(d)[1]
    print(f"{key}: {us:8.1f} us  {fl / us / 1e6:7.1f} TFLOP/s  plan {algos.fused_plan(d, 'tc3xbf16')['ctas']} ctas", flush=True)

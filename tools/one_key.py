"""Fused conv for one descriptor key, checked against torch fp64 (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import algos, harness
from paper_2407_10730_b200.descriptor import parse_key
for key in sys.argv[1:]:
    d = parse_key(key)
    inp = harness.device_inputs(d, harness.RunConfig())
    print(key, algos.fused_layout(d), algos.fused_plan(d), flush=True)
    y = algos.conv_fused(inp)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(inp.input.double(), inp.weights.double(), stride=(d.stride_h, d.stride_w),
                                     padding=(d.pad_h, d.pad_w), dilation=(d.dil_h, d.dil_w), groups=d.groups)
    print("   err", ((y.double() - ref).abs().max() / (d.in_channels // d.groups * d.k_h * d.k_w) ** 0.5).item(), flush=True)

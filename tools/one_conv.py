"""Run one fused conv (K3 + K0 + K6/K7) on a config once and check it (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from dataclasses import replace
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
d = CONFIGS[name]
if len(sys.argv) > 2:
    d = replace(d, batch=int(sys.argv[2]))
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.random((d.batch, d.in_channels, d.in_h, d.in_w), dtype=np.float32) * 2 - 1).cuda()
w = torch.from_numpy(rng.random((d.out_channels, d.in_channels, d.k_h, d.k_w), dtype=np.float32) * 2 - 1).cuda()
y = algos.conv_fused(algos.ConvInputs(desc=d, input=x, weights=w))
torch.cuda.synchronize()
ref = torch.nn.functional.conv2d(x.double(), w.double(), stride=d.stride_h, padding=d.pad_h)
err = (y.double() - ref).abs().max().item() / (d.in_channels * d.k_h * d.k_w) ** 0.5
print(name, d.batch, "layout", algos.fused_layout(d), "err", err)

"""cfg3 fused conv (K7, 3xBF16 and 3xTF32) and cfg4 Im2col-GEMM (K1 + K8) once each, after
warm-up (ncu target: 4 matching launches per round, 2 warm-up rounds)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device
from paper_2407_10730_b200.timing import PhaseLedger
i3 = to_device(make_inputs(CONFIGS["cfg3"], RunConfig(seed=0)))
i4 = to_device(make_inputs(CONFIGS["cfg4"], RunConfig(seed=0)))
for _ in range(3):  # two warm-up rounds, then the captured one
    algos.conv_fused(i3)
    algos.conv_fused(i3, variant="tc3xtf32")
    algos.conv_baseline_im2col_gemm(i4, PhaseLedger())
    torch.cuda.synchronize()
torch.cuda.synchronize()
print("ok")

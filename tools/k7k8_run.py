"""cfg3 fused conv (K7) and cfg4 Im2col-GEMM (K8) once each, after warm-up (ncu target)."""
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
for _ in range(2):
    algos.conv_fused(i3)
    algos.conv_baseline_im2col_gemm(i4, PhaseLedger())
torch.cuda.synchronize()
algos.conv_fused(i3)
algos.conv_baseline_im2col_gemm(i4, PhaseLedger())
torch.cuda.synchronize()
print("ok")

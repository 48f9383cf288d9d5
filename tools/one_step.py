"""One stepwise algorithm call on a config (diagnostics / ncu target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device
from paper_2407_10730_b200.timing import PhaseLedger
name, alg, v = (sys.argv[1:] + ["cfg4", "im2col", "tc3xbf16"][len(sys.argv) - 1:])[:3]
d = CONFIGS[name]
inp = to_device(make_inputs(d, RunConfig(seed=0)))
fn = algos.conv_baseline_im2col_gemm if alg == "im2col" else algos.conv_main_blocked_direct
for _ in range(3):
    fn(inp, PhaseLedger(), variant=v)
torch.cuda.synchronize()
print("ok")

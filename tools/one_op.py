"""Run one descriptor key through one path (diagnostics): python tools/one_op.py KEY MODE [variant]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import algos, harness
from paper_2407_10730_b200.descriptor import parse_key
from paper_2407_10730_b200.timing import EventLedger
key, mode = sys.argv[1], sys.argv[2]
variant = sys.argv[3] if len(sys.argv) > 3 else None
d = parse_key(key)
inp = harness.device_inputs(d, harness.RunConfig())
fn = {"fused": lambda: algos.conv_fused(inp, variant=variant or "auto"),
      "baseline": lambda: algos.conv_baseline_im2col_gemm(inp, EventLedger(), variant=variant or "tc3xtf32"),
      "main": lambda: algos.conv_main_blocked_direct(inp, EventLedger(), variant=variant or "tc3xtf32")}[mode]
for i in range(3):
    t = time.time()
    y = fn()
    torch.cuda.synchronize()
    print(key, mode, i, f"{(time.time() - t) * 1e3:.1f} ms", float(y.abs().max()), flush=True)

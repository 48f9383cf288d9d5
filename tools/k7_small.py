"""One small K7 (direct few-channel conv) launch checked against the oracle: the target of
compute-sanitizer runs (diagnostics).

    compute-sanitizer --tool memcheck python tools/k7_small.py
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.descriptor import parse_key
from paper_2407_10730_b200.harness import RunConfig, make_inputs
from paper_2407_10730_b200.tensor import normalized_max_err
from oracle import conv_oracle as orc

for key in sys.argv[1:] or ["n2_c3x64x64_f64x7x7_s2x2_p3x3_d1x1_g1_b1", "n1_c4x40x40_f32x3x3_s1x1_p1x1_d1x1_g1_b0"]:
    d = parse_key(key)
    assert algos.fused_layout(d, "tc3xbf16")["path"] == 2, key
    inp = make_inputs(d, RunConfig(seed=0))
    y = np.asarray(algos.conv_fused(inp, variant="tc3xbf16"))
    ref = orc.conv_direct_naive(d, np.asarray(inp.input), np.asarray(inp.weights),
                                None if inp.bias is None else np.asarray(inp.bias))
    print(key, "normalized max err", normalized_max_err(y, ref, d.in_channels // d.groups * d.k_h * d.k_w))

# K7: is the A build bound by the F2FP conversions?  hi by truncation (PRMT) vs conversion.
mkdir -p gpurun_out/r2az _ab
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=1','-DCB_TS_TRUNC_HI'), out='_ab/k1t.so')" > gpurun_out/r2az/b1.log 2>&1 || echo fail
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=3','-DCB_TS_TRUNC_HI'), out='_ab/k3t.so')" > gpurun_out/r2az/b3.log 2>&1 || echo fail
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=1',), out='_ab/k1.so')" > gpurun_out/r2az/b1n.log 2>&1 || echo fail
for rep in 1 2; do
for l in k1 k1t k3t; do echo "$l: $(CB_LIB_PATH=_ab/$l.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done
done
CB_LIB_PATH=_ab/k1t.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs" 2>&1 | tail -2
CB_LIB_PATH=_ab/k1t.so CB_TS_TRACE=0 python - <<'PY'
import numpy as np, torch
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs
from paper_2407_10730_b200.tensor import normalized_max_err
from oracle import conv_oracle
inp = make_inputs(CONFIGS["cfg3"], RunConfig(seed=0))
y = algos.conv_fused(inp)
ref = conv_oracle.conv_im2col64(inp) if hasattr(conv_oracle, "conv_im2col64") else None
print("cfg3 trunc-hi normalized err", normalized_max_err(np.asarray(y), ref, CONFIGS["cfg3"]) if ref is not None else "n/a")
PY

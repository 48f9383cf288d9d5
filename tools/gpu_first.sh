set -x
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv
timeout 120 python -c "
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, torch
from corpus import corpus
from oracle import conv_oracle as orc
from paper_2407_10730_b200.algos import ConvInputs, conv_fused
d=corpus(3,seed=7)[0]; x,w,b=orc.make_inputs(d)
inp=ConvInputs(desc=d,input=x,weights=w,bias=b)
ref=orc.conv_direct_naive(d,x,w,b)
for v in ('ffma','tc3xtf32','tc3xbf16'):
    y=conv_fused(inp,variant=v); print(v, orc.normalized_max_err(y,ref,orc.reduction_len(d)), flush=True)
" > gpurun_out/first_small.log 2>&1; echo "small rc=$?"
cat gpurun_out/first_small.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -s > gpurun_out/first_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/first_pytest.log
timeout 300 python tools/devtime.py > gpurun_out/first_devtime.log 2>&1; echo "devtime rc=$?"
cat gpurun_out/first_devtime.log

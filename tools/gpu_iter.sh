# one GPU iteration: small smoke, parity suite, dev timings (each bounded by timeout)
set -o pipefail
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 120 python -c "
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
from corpus import corpus, cfg
from oracle import conv_oracle as orc
from paper_2407_10730_b200.algos import ConvInputs, conv_fused, fused_layout
for d in corpus(4,seed=7)[:3] + [cfg('cfg1'), cfg('cfg3', batch=1)]:
    x,w,b=orc.make_inputs(d); inp=ConvInputs(desc=d,input=x,weights=w,bias=b)
    ref=orc.conv_im2col64(d,x,w,b)
    for v in ('tc3xtf32','tc3xbf16'):
        y=conv_fused(inp,variant=v); print(v, fused_layout(d,v)['path'], orc.normalized_max_err(y,ref,orc.reduction_len(d)), flush=True)
" 2>&1 | tail -20; echo "small rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -s 2>&1 | tail -25; echo "pytest rc=$?"
timeout 300 python tools/devtime.py $DEVTIME_CFGS 2>&1 | tail -40; echo "devtime rc=$?"
timeout 120 python tools/devtime.py acc 2>&1 | tail -10

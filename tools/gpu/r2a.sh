mkdir -p gpurun_out/r2a
(nproc; lscpu | head -30; free -g; cat /proc/cpuinfo | grep "model name" | head -1) > gpurun_out/r2a/host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2a/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2a/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo "bench rc=$?"
python - <<'PY' > gpurun_out/r2a/bench_oracle_time.txt 2>&1
import time, numpy as np, sys
sys.path.insert(0,'.')
from oracle import conv_oracle as orc
from paper_2407_10730_b200.configs import CONFIGS
from dataclasses import replace
for n in ["cfg4","cfg3"]:
    d=CONFIGS[n]
    t=time.time(); x,w,b=orc.make_inputs(d,0); t1=time.time()
    y=orc.conv_im2col64(d,x,w,b); t2=time.time()
    print(n,"gen",t1-t,"oracle",t2-t1, flush=True)
a=np.random.rand(4096,4096); t=time.time(); a@a; print("dgemm 4096 GF/s", 2*4096**3/(time.time()-t)/1e9)
PY

# one GPU iteration: parity suite, dev timings (each bounded by timeout)
set -o pipefail
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15; echo "pytest rc=$?"
for CG in 1 2; do CB_TMA_CG=$CG timeout 300 python tools/devtime.py cfg4 2>&1 | grep fused; done
timeout 300 python tools/devtime.py cfg3 cfg1 2>&1 | grep -v plan= ; true
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print({k: d[k] for k in ('value','ms_per_step','gpu_launches','step_phases_us','clocks')}); print(d['roofline']); print(d['e2e'])
print({k:(v['operation_us'], v['pack_share']) for k,v in d['breakdown'].items()})"

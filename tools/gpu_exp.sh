set -o pipefail
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print({k: d[k] for k in ('value','ms_per_step','gpu_launches','step_phases_us','clocks')}); print(d['roofline']); print(d['e2e'])
print({k:(round(v['operation_us'],1), round(v['pack_share'],3)) for k,v in d['breakdown'].items()})"

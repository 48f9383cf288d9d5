set -o pipefail
mkdir -p gpurun_out/r2an
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2an/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2an/pytest.log
timeout 300 python tools/ktime.py pack cfg1 cfg2a cfg2b cfg3 cfg4 2>&1 | tail -10
timeout 900 python bench.py --no-cpu-baseline --no-variants > gpurun_out/r2an/bench.json 2> gpurun_out/r2an/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2an/bench.json').read().splitlines()[-1])
print(d['value'], d['ms_per_step'])
for c,row in d['configs'].items():
    print(c, {k:(round(v['operation_us'],1), {p:round(t,1) for p,t in v['phases_us'].items() if p in ('pre_reorder','in_packing','in_microkernel')}) for k,v in row.items() if k in ('im2col_gemm','sconv')})
PY

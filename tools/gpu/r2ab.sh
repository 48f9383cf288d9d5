set -o pipefail
mkdir -p gpurun_out/r2ab
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2ab/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ab/pytest.log
for a in "cfg4 im2col" "cfg4 sconv" "cfg3 im2col" "cfg3 sconv"; do for env in "CB_K8_NO_TMA_STORE=1" "CB_X=0"; do echo "== $a $env"; env $env timeout 120 python tools/k8_trace.py $a tc3xbf16 2>&1 | grep -E "CTAs;|item [01]"; done; done > gpurun_out/r2ab/k8.log 2>&1; cat gpurun_out/r2ab/k8.log
timeout 900 python bench.py --no-cpu-baseline --no-variants > gpurun_out/r2ab/bench.json 2> gpurun_out/r2ab/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2ab/bench.json').read().splitlines()[-1])
print(d['value'], d['ms_per_step'])
for c,row in d['configs'].items():
    print(c, {k:(round(v['operation_us'],1), round(v['phases_us'].get('in_microkernel',0),1)) for k,v in row.items()})
PY

mkdir -p gpurun_out/r2bu
SECONDS=0; timeout 900 python bench.py > gpurun_out/r2bu/bench.json 2> gpurun_out/r2bu/bench.err; echo "bench rc=$?"
echo "bench wall ${SECONDS}s"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2bu/bench.json').read().strip().splitlines()[-1])
print(json.dumps(d['targets'], indent=1))
print(d['value'], d['roofline']['frac'])
PY

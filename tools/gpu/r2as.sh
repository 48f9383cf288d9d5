# Session re-entry check: GPU tests, smoke, default bench line, reference arm, K7 device times on cfg3.
set -o pipefail
mkdir -p gpurun_out/r2as
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2as/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2as/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2as/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2as/smoke.log
timeout 600 python bench.py > gpurun_out/r2as/bench.json 2> gpurun_out/r2as/bench.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.loads(open("gpurun_out/r2as/bench.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","e2e","roofline","clocks")})
PY
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2as/bench_ref.json 2> gpurun_out/r2as/bench_ref.err; echo "ref rc=$?"
tail -c 600 gpurun_out/r2as/bench_ref.json
timeout 300 python tools/ktime.py cfg3 > gpurun_out/r2as/ktime_cfg3.log 2>&1; tail -5 gpurun_out/r2as/ktime_cfg3.log
CB_KT_COLD=1 timeout 300 python tools/ktime.py cfg3 > gpurun_out/r2as/ktime_cfg3_cold.log 2>&1; tail -5 gpurun_out/r2as/ktime_cfg3_cold.log

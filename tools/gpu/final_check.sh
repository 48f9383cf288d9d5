# Final-state check: GPU tests, smoke, default bench line, reference arm.
set -o pipefail
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/final/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final/smoke.log
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/final/bench.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","clocks")}, d["roofline"]["frac"], d["e2e"]["value"], d["targets"]["fused_conv_roofline_frac"], d["parity"]["max_err"])
r=json.loads(open("gpurun_out/final/bench_ref.json").read().strip().splitlines()[-1])
print(r.get("value"), r.get("unit"), r.get("ms_per_step"), r.get("impl"))
PY

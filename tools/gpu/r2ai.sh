set -o pipefail
mkdir -p gpurun_out/r2ai
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2ai/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ai/pytest.log
timeout 600 python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs
d = CONFIGS["cfg4"]
h = make_inputs(d, RunConfig(seed=0))
for _ in range(2):
    print(json.dumps(bench.e2e_dropin(d, "tc3xbf16", h.input, h.weights)))
PY

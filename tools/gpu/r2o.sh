set -o pipefail
mkdir -p gpurun_out/r2o
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r2o/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2o/pytest.log
for env in "CB_K8_DEBUG=0" "CB_K8_DEBUG=15" "CB_K8_DEBUG=4"; do echo "== $env"; env $env timeout 120 python tools/k8_trace.py cfg4 im2col tc3xbf16 2>&1 | grep -E "CTAs;|item|pace"; done > gpurun_out/r2o/k8.log 2>&1; cat gpurun_out/r2o/k8.log
for a in "cfg4 sconv tc3xbf16" "cfg4 im2col tc3xtf32" "cfg3 im2col tc3xbf16"; do timeout 120 python tools/k8_trace.py $a 2>&1 | grep -E "CTAs;|item|pace"; done >> gpurun_out/r2o/k8.log 2>&1; tail -14 gpurun_out/r2o/k8.log

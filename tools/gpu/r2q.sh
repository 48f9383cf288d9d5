set -o pipefail
mkdir -p gpurun_out/r2q
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2q/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2q/pytest.log
for a in "cfg4 im2col tc3xbf16" "cfg4 sconv tc3xbf16" "cfg4 im2col tc3xtf32"; do timeout 120 python tools/k8_trace.py $a 2>&1 | grep -E "CTAs;|item|pace"; done > gpurun_out/r2q/k8.log 2>&1; cat gpurun_out/r2q/k8.log
CB_K8_NSPLIT=1 timeout 120 python tools/k8_trace.py cfg4 im2col tc3xbf16 2>&1 | grep -E "CTAs;|item"

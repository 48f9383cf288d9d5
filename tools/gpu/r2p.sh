set -o pipefail
mkdir -p gpurun_out/r2p
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2p/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2p/pytest.log
for a in "cfg4 im2col tc3xbf16" "cfg4 sconv tc3xbf16" "cfg4 im2col tc3xtf32" "cfg3 im2col tc3xbf16"; do timeout 120 python tools/k8_trace.py $a 2>&1 | grep -E "CTAs;|item|pace"; done > gpurun_out/r2p/k8.log 2>&1; cat gpurun_out/r2p/k8.log

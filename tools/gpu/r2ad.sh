set -o pipefail
mkdir -p gpurun_out/r2ad
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2ad/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ad/pytest.log
for a in "cfg4 im2col tc3xbf16" "cfg4 im2col tc3xtf32"; do for env in "CB_X=0" "CB_K8_KSPLIT=2" "CB_K8_KSPLIT=3"; do echo "== $a $env"; env $env timeout 120 python tools/k8_trace.py $a 2>&1 | grep -E "CTAs;|item [01]|rror"; done; done > gpurun_out/r2ad/k8.log 2>&1; cat gpurun_out/r2ad/k8.log

set -o pipefail
mkdir -p gpurun_out/r2r
for env in "CB_K8_KPARTS=2" "CB_K8_KPARTS=3" "CB_K8_NSPLIT=1" "CB_K8_KPARTS=2" "CB_K8_NSPLIT=1"; do echo "== $env"; env $env timeout 120 python tools/k8_trace.py cfg4 im2col tc3xbf16 2>&1 | grep -E "CTAs;|item"; done > gpurun_out/r2r/k8.log 2>&1; cat gpurun_out/r2r/k8.log

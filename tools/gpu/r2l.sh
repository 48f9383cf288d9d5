set -o pipefail
mkdir -p gpurun_out/r2l
for env in "CB_K8_DEBUG=0" "CB_K8_DEBUG=1" "CB_K8_DEBUG=2" "CB_K8_DEBUG=3" "CB_K8_ASTAGES=6" "CB_K8_ASTAGES=2 CB_K8_BSTAGES=3"; do echo "== $env"; env $env timeout 120 python tools/k8_trace.py cfg4 im2col tc3xbf16 2>&1 | grep -E "CTAs;|item|pace"; done > gpurun_out/r2l/k8.log 2>&1; cat gpurun_out/r2l/k8.log

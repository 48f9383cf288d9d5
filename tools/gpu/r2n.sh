set -o pipefail
mkdir -p gpurun_out/r2n
for env in "CB_K8_DEBUG=0" "CB_K8_DEBUG=4" "CB_K8_DEBUG=8" "CB_K8_DEBUG=11" "CB_K8_DEBUG=15" "CB_K8_BN=128" "CB_K8_BN=64"; do echo "== $env"; env $env timeout 120 python tools/k8_trace.py cfg4 im2col tc3xbf16 2>&1 | grep -E "CTAs;|item 0|pace"; done > gpurun_out/r2n/k8.log 2>&1; cat gpurun_out/r2n/k8.log

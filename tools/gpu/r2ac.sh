set -o pipefail
mkdir -p gpurun_out/r2ac
for a in "cfg4 im2col" "cfg4 sconv" "cfg3 im2col"; do for env in "CB_K8_NO_TMA_STORE=1" "CB_X=0"; do echo "== $a $env"; env $env timeout 120 python tools/k8_trace.py $a tc3xbf16 2>&1 | grep -E "CTAs;|item [01]|rror"; done; done > gpurun_out/r2ac/k8.log 2>&1; cat gpurun_out/r2ac/k8.log

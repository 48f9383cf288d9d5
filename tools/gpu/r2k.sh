# K8 chunk-level trace, A stage count sweep; K7 full ncu capture
set -o pipefail
mkdir -p gpurun_out/r2k
timeout 120 python tools/k8_trace.py cfg4 im2col tc3xbf16 > gpurun_out/r2k/k8_trace.log 2>&1; cat gpurun_out/r2k/k8_trace.log
for s in 2 6 8; do echo "== CB_K8_ASTAGES=$s"; CB_K8_ASTAGES=$s timeout 120 python tools/k8_trace.py cfg4 im2col tc3xbf16 2>&1 | grep -E "CTAs;|item 0|pace"; done > gpurun_out/r2k/k8_astages.log 2>&1; cat gpurun_out/r2k/k8_astages.log
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:conv_ts_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r2k/k7_full -f python tools/k7k8_run.py > gpurun_out/r2k/ncu_k7.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r2k/ncu_k7.log

set -o pipefail
mkdir -p gpurun_out/r2al
for env in "CB_NO_ACT_FLAGS=1" "CB_X=0"; do echo "== $env"; env $env CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg4 2>&1 | tail -1; done
timeout 300 ncu --kernel-name regex:"act_split_flag" --launch-skip 3 --launch-count 1 --clock-control none --set full -o gpurun_out/r2al/k0f -f python tools/ktime.py cfg4 > /dev/null 2>&1; echo "ncu rc=$?"

set -o pipefail
mkdir -p gpurun_out/prof
CMD="python tools/ktime.py pack cfg4"
timeout 300 $CMD > gpurun_out/prof/pack_plain.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:im2col_band -s 3 -c 1 -o gpurun_out/prof/full_pack_cfg4 -f $CMD > gpurun_out/prof/ncu_pack.log 2>&1; echo "ncu rc=$?"

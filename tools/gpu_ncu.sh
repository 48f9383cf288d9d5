# One ncu --set full capture of the bench step's kernels (after the plain run exits 0).
set -o pipefail
mkdir -p gpurun_out/prof
CMD="python bench.py --no-breakdown --no-cpu-baseline --steps 2 --warmup 3"
timeout 300 $CMD > gpurun_out/prof/plain.json 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tma|act_split|weight_split_taps" -s 3 -c 3 -o gpurun_out/prof/full_step -f $CMD > gpurun_out/prof/ncu_full.log 2>&1; echo "ncu rc=$?"

# ncu evidence for profiles/: launch list of the bench command + full captures
set -o pipefail
mkdir -p gpurun_out/prof
CMD="python bench.py --steps 4 --warmup 2 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/prof/plain.json 2> gpurun_out/prof/plain.err; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches.csv $CMD > gpurun_out/prof/ncu_launch.log 2>&1; echo "launch-list rc=$?"
for k in conv_tma act_split weight_split_taps im2col_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof/full_$k $CMD > gpurun_out/prof/ncu_$k.log 2>&1; echo "full $k rc=$?"
done
ls -la gpurun_out/prof

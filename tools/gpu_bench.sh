# bench + ncu launch list + one full ncu capture of the top kernel
set -o pipefail
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 6000; echo
SHORT="python bench.py --steps 2 --warmup 1 --no-breakdown --no-cpu-baseline"
timeout 300 $SHORT > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
timeout 300 $SHORT > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tma -s 1 -c 1 \
    -o gpurun_out/prof_conv_tma $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
tail -5 gpurun_out/ncu_full.log

set -o pipefail
SHORT="python bench.py --steps 2 --warmup 1 --no-breakdown --no-cpu-baseline"
timeout 300 $SHORT > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tma -s 1 -c 1 \
    -o gpurun_out/prof_conv_tma_cg2 $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
CB_TMA_CG=1 CB_TMA_BN=128 timeout 300 $SHORT > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
CB_TMA_CG=1 CB_TMA_BN=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tma -s 1 -c 1 \
    -o gpurun_out/prof_conv_tma_cg1 $SHORT > gpurun_out/ncu_full1.log 2>&1; echo "ncu-full1 rc=$?"

set -o pipefail
mkdir -p gpurun_out/r2x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_few or baseline_configs or known or model_layers or sweep_plan" > gpurun_out/r2x/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2x/pytest.log
for r in 1 2; do CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1; done > gpurun_out/r2x/k7.log 2>&1; cat gpurun_out/r2x/k7.log
for b in 2 8 32; do echo "== N=$b"; CB_KT_BATCH=$b timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1; done >> gpurun_out/r2x/k7.log 2>&1; tail -6 gpurun_out/r2x/k7.log
timeout 300 ncu --kernel-name regex:"conv_ts_kernel" --launch-skip 2 --launch-count 1 --clock-control none --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_sample_count --csv python tools/k7k8_run.py > gpurun_out/r2x/ncu.csv 2>/dev/null; echo "ncu rc=$?"

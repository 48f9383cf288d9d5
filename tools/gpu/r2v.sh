set -o pipefail
mkdir -p gpurun_out/r2v
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_few or planes or baseline_configs or known" > gpurun_out/r2v/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2v/pytest.log
for env in "CB_TS_NO_PLANES=1" "CB_TS_X=0" "CB_TS_NO_PLANES=1" "CB_TS_X=0"; do echo "== $env"; env $env CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1; done > gpurun_out/r2v/k7.log 2>&1; cat gpurun_out/r2v/k7.log
for b in 2 8 32; do echo "== N=$b"; CB_KT_BATCH=$b timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1; done >> gpurun_out/r2v/k7.log 2>&1; tail -6 gpurun_out/r2v/k7.log
timeout 300 ncu --kernel-name regex:"conv_tsp?_kernel" --launch-skip 2 --launch-count 1 --clock-control none --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,lts__t_bytes.sum --csv python tools/k7k8_run.py > gpurun_out/r2v/ncu.csv 2>/dev/null; echo "ncu rc=$?"

# K7 (cfg3): pair vs single CTA, TMA-store vs direct epilogue, bottleneck switches; parity of
mkdir -p gpurun_out/r2e
timeout 400 python tools/sweep.py --min-gflop 20 --max-gflop 45 --warmups 1 --runs 2 --verbose --out gpurun_out/r2e/sw > gpurun_out/r2e/sw.log 2>&1; echo "sweep20-45 rc=$?"; tail -3 gpurun_out/r2e/sw.log
# the K7 variants; the new bench line; K7 smem counters.
mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_few_channel or baseline_configs_all_paths or known_answers" > gpurun_out/r2e/pytest_k7.log 2>&1; echo "pytest(pair) rc=$?"; tail -2 gpurun_out/r2e/pytest_k7.log
for env in "CB_TS_CG=1" "CB_TS_CG=1 CB_TS_NO_TMA_STORE=1" "CB_TS_CG=2" "CB_TS_CG=2 CB_TS_NO_TMA_STORE=1" "CB_TS_CG=1 CB_TS_DEBUG=8" "CB_TS_CG=1 CB_TS_DEBUG=1" "CB_TS_CG=1 CB_TS_DEBUG=16" "CB_TS_CG=1 CB_TS_DEBUG=4" "CB_TS_CG=2 CB_TS_DEBUG=8" "CB_TS_CG=2 CB_TS_DEBUG=16"; do
  echo "== $env"; env $env timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1
done > gpurun_out/r2e/k7.log 2>&1; cat gpurun_out/r2e/k7.log
CB_TS_CG=1 timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_few_channel" > gpurun_out/r2e/pytest_k7_cg1.log 2>&1; echo "pytest(cg1) rc=$?"; tail -1 gpurun_out/r2e/pytest_k7_cg1.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e/bench.json 2> gpurun_out/r2e/bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r2e/bench.json; tail -3 gpurun_out/r2e/bench.err
timeout 600 ncu --kernel-name regex:conv_ts_kernel --launch-skip 2 --launch-count 1 --clock-control none \
  --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__cycles_active.avg,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active \
  --csv python tools/k7k8_run.py > gpurun_out/r2e/ncu_k7_smem.csv 2> gpurun_out/r2e/ncu_k7.err; echo "ncu rc=$?"

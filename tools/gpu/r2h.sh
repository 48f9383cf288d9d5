# K0/K3 after the occupancy/unrolled-load fixes; K7 variants (warm and L2-cold); K7 smem counters
set -o pipefail
mkdir -p gpurun_out/r2h
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or baseline_configs or direct_few" > gpurun_out/r2h/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2h/pytest.log
for c in cfg4 cfg3; do CB_KT_COLD=1 timeout 120 python tools/ktime.py $c 2>&1 | tail -2; done > gpurun_out/r2h/ktime.log 2>&1; cat gpurun_out/r2h/ktime.log
timeout 300 python bench.py --no-breakdown --no-cpu-baseline --no-variants > gpurun_out/r2h/bench_plain.json 2> gpurun_out/r2h/bench_plain.err; echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2h/bench_plain.json').read().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['step_phases_us'])"
for env in "CB_TS_CG=1" "CB_TS_NO_TMA_STORE=1" "CB_TS_CG=2" "CB_TS_NO_PAIR=1" "CB_TS_DEBUG=8" "CB_TS_DEBUG=1" "CB_TS_DEBUG=16" "CB_TS_DEBUG=4" "CB_TS_DEBUG=24" "CB_TS_DEBUG=9"; do
  echo "== $env"; env $env CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1
done > gpurun_out/r2h/k7.log 2>&1; cat gpurun_out/r2h/k7.log
M=gpu__time_duration.sum,sm__cycles_elapsed.max,l1tex__data_bank_reads.sum,l1tex__data_bank_writes.sum,l1tex__data_pipe_tc_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_cmd_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_cmd_write.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --kernel-name regex:"conv_ts_kernel|gemm_ts_kernel" --launch-skip 4 --launch-count 2 --clock-control none --metrics $M --csv python tools/k7k8_run.py > gpurun_out/r2h/ncu_k7k8_smem.csv 2> gpurun_out/r2h/ncu.err; echo "ncu rc=$?"

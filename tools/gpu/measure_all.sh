# Round-2 measurement set: GPU tests, smoke, bench line, reference arm, launch list of the
# bench command, ncu --set full of the step's kernels and of K7 / K8.
set -o pipefail
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/prof/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/prof/pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/prof/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/prof/smoke.log
timeout 900 python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof/bench_ref.json 2> gpurun_out/prof/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --no-breakdown --no-cpu-baseline --no-variants --steps 5 --warmup 3"
timeout 300 $CMD > gpurun_out/prof/bench_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv $CMD > gpurun_out/prof/ncu_launches.log 2>&1; echo "launches rc=$?"
CMD2="python bench.py --no-breakdown --no-cpu-baseline --no-variants --steps 2 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_tma|act_split|weight_split_taps" -s 3 -c 3 -o gpurun_out/prof/full_step -f $CMD2 > gpurun_out/prof/ncu_full.log 2>&1; echo "ncu step rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_ts_kernel|gemm_ts_kernel|im2col_band" -s 8 -c 4 -o gpurun_out/prof/full_k7k8 -f python tools/k7k8_run.py > gpurun_out/prof/ncu_k7k8.log 2>&1; echo "ncu k7k8 rc=$?"

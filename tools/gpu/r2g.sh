# Round 2 re-entry: GPU tests, smoke, bench line, reference arm, launch list of the bench command.
set -o pipefail
mkdir -p gpurun_out/r2g
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2g/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2g/pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2g/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2g/smoke.log
timeout 900 python bench.py > gpurun_out/r2g/bench.json 2> gpurun_out/r2g/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2g/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2g/bench_ref.json 2> gpurun_out/r2g/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/r2g/bench_ref.json
CMD="python bench.py --no-breakdown --no-cpu-baseline --no-variants --steps 5 --warmup 3"
timeout 300 $CMD > gpurun_out/r2g/bench_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g/launches.csv $CMD > gpurun_out/r2g/ncu_launches.log 2>&1; echo "launches rc=$?"

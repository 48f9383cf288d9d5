# Round-end style measurement: bench line, reference arm, launch list of the bench command.
set -o pipefail
mkdir -p gpurun_out/prof
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.json
CMD="python bench.py --no-breakdown --no-cpu-baseline --steps 5 --warmup 3"
timeout 300 $CMD > gpurun_out/prof/bench_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv $CMD > gpurun_out/prof/ncu_launches.log 2>&1; echo "launches rc=$?"

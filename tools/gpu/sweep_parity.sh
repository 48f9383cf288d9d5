# After the K7 mixed-layout / single-producer changes: the full config-5 sweep on make_inputs
# data with CPU-oracle parity on every op, the reference convbench report and the speedup chart.
set -o pipefail
mkdir -p gpurun_out/sweep
timeout 3000 python tests/sweep_parity.py --warmups 1 --runs 3 --pending 24 --out gpurun_out/sweep/sweep9243 > gpurun_out/sweep/sweep.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/sweep/sweep.log
PYTHONPATH=baseline/_ref timeout 300 python -m convbench.cli report --main gpurun_out/sweep/sweep9243/results_main.csv --baseline gpurun_out/sweep/sweep9243/results_baseline.csv --out-speedup gpurun_out/sweep/sweep9243/ref_speedup.csv --out-breakdown gpurun_out/sweep/sweep9243/ref_breakdown.csv --out-summary gpurun_out/sweep/sweep9243/ref_summary.json > gpurun_out/sweep/report.log 2>&1; echo "report rc=$?"; tail -3 gpurun_out/sweep/report.log
python tools/charts.py speedup --in gpurun_out/sweep/sweep9243/ref_speedup.csv --out gpurun_out/sweep/sweep9243/speedup.svg --sort by-speedup --log-y; echo "chart rc=$?"

# Full config-5 sweep on make_inputs data with CPU-oracle parity on every op (after the K8
# schedule rewrite and the 3xBF16 stepwise default), then the reference convbench report.
mkdir -p gpurun_out/r2ae
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r2ae/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ae/pytest.log
timeout 3000 python tests/sweep_parity.py --warmups 1 --runs 3 --pending 24 --out gpurun_out/r2ae/sweep9243 > gpurun_out/r2ae/sweep.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/r2ae/sweep.log
PYTHONPATH=baseline/_ref timeout 300 python -m convbench.cli report --main gpurun_out/r2ae/sweep9243/results_main.csv --baseline gpurun_out/r2ae/sweep9243/results_baseline.csv --out-speedup gpurun_out/r2ae/sweep9243/ref_speedup.csv --out-breakdown gpurun_out/r2ae/sweep9243/ref_breakdown.csv --out-summary gpurun_out/r2ae/sweep9243/ref_summary.json > gpurun_out/r2ae/report.log 2>&1; echo "report rc=$?"; tail -3 gpurun_out/r2ae/report.log
python tools/charts.py speedup --in gpurun_out/r2ae/sweep9243/ref_speedup.csv --out gpurun_out/r2ae/sweep9243/speedup.svg --sort by-speedup --log-y; echo "chart rc=$?"

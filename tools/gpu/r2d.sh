# Full config-5 sweep on make_inputs data with CPU-oracle parity on every op, then the
# unmodified reference `convbench report` on the results CSVs.
mkdir -p gpurun_out/r2d
df -h /dev/shm > gpurun_out/r2d/shm.txt 2>&1
timeout 4200 python tests/sweep_parity.py --warmups 2 --runs 5 --pending 16 --out gpurun_out/r2d/sweep9243 > gpurun_out/r2d/sweep.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/r2d/sweep.log
PYTHONPATH=baseline/_ref timeout 600 python -m convbench.cli report --main gpurun_out/r2d/sweep9243/results_main.csv --baseline gpurun_out/r2d/sweep9243/results_baseline.csv --out-speedup gpurun_out/r2d/sweep9243/ref_speedup.csv --out-breakdown gpurun_out/r2d/sweep9243/ref_breakdown.csv --out-summary gpurun_out/r2d/sweep9243/ref_summary.json > gpurun_out/r2d/report.log 2>&1; echo "report rc=$?"; tail -3 gpurun_out/r2d/report.log

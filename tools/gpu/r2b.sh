mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b/pytest.log
timeout 900 python tests/sweep_parity.py --sample 300 --warmups 1 --runs 2 --out gpurun_out/r2b/sweep300 > gpurun_out/r2b/sweep.log 2>&1; echo "sweep rc=$?"; tail -5 gpurun_out/r2b/sweep.log

mkdir -p gpurun_out/r2c
timeout 600 python tools/promote_probe.py 0 2048 4096 > gpurun_out/r2c/probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/r2c/probe.log | tail -30
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "large_reductions or sweep_plan or tail_split or many_k" > gpurun_out/r2c/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2c/pytest.log

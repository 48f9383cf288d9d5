mkdir -p gpurun_out/r2c
timeout 600 python tools/promote_probe.py > gpurun_out/r2c/probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/r2c/probe.log | tail -30

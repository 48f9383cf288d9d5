# K7 change check: parity tests that reach K7, device time on cfg3, per-tile trace.
mkdir -p gpurun_out/r2av
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs or model_layers or sweep_plan" > gpurun_out/r2av/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2av/pytest.log
timeout 300 python tools/ktime.py cfg3 > gpurun_out/r2av/ktime_cfg3.log 2>&1; tail -1 gpurun_out/r2av/ktime_cfg3.log
CB_KT_COLD=1 timeout 300 python tools/ktime.py cfg3 > gpurun_out/r2av/ktime_cfg3_cold.log 2>&1; tail -1 gpurun_out/r2av/ktime_cfg3_cold.log
CB_TS_TRACE=1 timeout 900 python tools/ts_trace.py cfg3 > gpurun_out/r2av/ts_trace.log 2>&1; echo "rc=$?"
sed -n 1,16p gpurun_out/r2av/ts_trace.log

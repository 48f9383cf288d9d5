mkdir -p gpurun_out/r2bd
CB_TS_TRACE=1 timeout 900 python tools/ts_trace.py cfg3 > gpurun_out/r2bd/ts_trace.log 2>&1; echo "rc=$?"
sed -n 1,16p gpurun_out/r2bd/ts_trace.log

# K7 per-tile trace on cfg3 (diagnostics build compiled on the box).
mkdir -p gpurun_out/k7_trace
CB_TS_TRACE=1 timeout 900 python tools/ts_trace.py cfg3 > gpurun_out/k7_trace/ts_trace.log 2>&1; echo "rc=$?"
tail -30 gpurun_out/k7_trace/ts_trace.log

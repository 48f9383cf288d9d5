# K8 per-item timelines on cfg4 (Im2col-GEMM and SConv, 3xBF16)
mkdir -p gpurun_out/r2aq
for p in im2col sconv; do timeout 300 python tools/k8_trace.py cfg4 $p tc3xbf16 2>&1 | tail -14; done > gpurun_out/r2aq/trace.log 2>&1; cat gpurun_out/r2aq/trace.log

mkdir -p gpurun_out/bench_table
SECONDS=0
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_table/bench.json 2> gpurun_out/bench_table/bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/bench_table/bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_table/bench.json').read().strip().splitlines()[-1])
for c,v in d['configs'].items():
    for p,q in v.items():
        extra = {k: round(q[k], 3) for k in ('kernel_alone_us', 'kernel_alone_roofline_frac', 'pack_alone_us', 'pack_alone_hbm_frac') if q.get(k)}
        print(c, p, q['variant'], 'op events', round(q['operation_us'], 1), 'op alone', round(q['operation_alone_us'], 1), 'GFLOP/s', round(q['gflops_alone']), extra)
PY

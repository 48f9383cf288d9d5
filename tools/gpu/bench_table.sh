mkdir -p gpurun_out/bench_table
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_table/bench.json 2> gpurun_out/bench_table/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_table/bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_table/bench.json').read().strip().splitlines()[-1])
for c,v in d['configs'].items():
    for p,q in v.items():
        if 'kernel_alone_us' in q: print(c,p,q['variant'],'phase',round(q['kernel_us'],1),'alone',round(q['kernel_alone_us'],1),'frac',round(q['kernel_alone_roofline_frac'],3), q['target_60pct_met'])
        if 'pack_alone_us' in q: print(c,p,q['pack_kernel'],'phase GB/s',round(q['pack_gbs']),'alone us',round(q['pack_alone_us'],1),'frac',round(q['pack_alone_hbm_frac'],3))
PY

# A stratified sample of the config-5 sweep through the fused path with the 3xTF32 split
# (K6 tf32, and the tf32 K7 on the few-channel ops), CPU-oracle parity on every op.
mkdir -p gpurun_out/sweep_tf32
timeout 1500 python tests/sweep_parity.py --sample 1500 --modes fused --fused-variant tc3xtf32 --warmups 1 --runs 2 --pending 24 --out gpurun_out/sweep_tf32/s > gpurun_out/sweep_tf32/sweep.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
s=json.load(open('gpurun_out/sweep_tf32/s/summary.json'))
v=s['modes']['fused']; p=v['parity']
print(s['ops_run'], v['status'], 'checked', p['checked'], 'over', p['over_gate'], 'max', p['max_err'], p['worst_op'])
PY

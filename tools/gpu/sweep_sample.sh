mkdir -p gpurun_out/sweep_bf16s
timeout 1500 python tests/sweep_parity.py --sample 2000 --warmups 1 --runs 2 --pending 24 --out gpurun_out/sweep_bf16s/s > gpurun_out/sweep_bf16s/sweep.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
s=json.load(open('gpurun_out/sweep_bf16s/s/summary.json'))
for m,v in s['modes'].items():
    p=v['parity']; print(m, v['status'], 'checked', p['checked'], 'over', p['over_gate'], 'max', p['max_err'])
PY

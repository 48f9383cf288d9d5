set -o pipefail
mkdir -p gpurun_out/r2ak
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2ak/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2ak/pytest.log
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
for env in "CB_NO_ACT_FLAGS=1" "CB_X=0" "CB_NO_ACT_FLAGS=1" "CB_X=0"; do env $env timeout 300 python bench.py --no-breakdown --no-cpu-baseline --no-variants > gpurun_out/r2ak/b.json 2>gpurun_out/r2ak/b.err; echo "rc=$?"; python -c "import json,sys;d=json.loads(open('gpurun_out/r2ak/b.json').read().splitlines()[-1]);print('$env',round(d['value']),d['ms_per_step'],d['step_phases_us'], d['e2e']['value'], d.get('parity'))"; done

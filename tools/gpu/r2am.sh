set -o pipefail
mkdir -p gpurun_out/r2am
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2am/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2am/pytest.log
for env in "CB_X=0" "CB_ACT_FLAGS=1" "CB_X=0" "CB_ACT_FLAGS=1"; do env $env timeout 300 python bench.py --no-breakdown --no-cpu-baseline --no-variants > gpurun_out/r2am/b.json 2>gpurun_out/r2am/b.err; python -c "import json,sys;d=json.loads(open('gpurun_out/r2am/b.json').read().splitlines()[-1]);print('$env',round(d['value']),d['ms_per_step'],d['step_phases_us'], d['e2e']['value'])"; done
CB_ACT_FLAGS=1 CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg4 2>&1 | tail -1

set -o pipefail
mkdir -p gpurun_out/r2aj
CB_TMA_LASTW=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or baseline_configs or tma_store" > gpurun_out/r2aj/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2aj/pytest.log
for env in "CB_X=0" "CB_TMA_LASTW=1" "CB_X=0" "CB_TMA_LASTW=1"; do echo "== $env"; env $env CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg4 2>&1 | tail -1; done > gpurun_out/r2aj/k6.log 2>&1; cat gpurun_out/r2aj/k6.log
for env in "CB_X=0" "CB_TMA_LASTW=1" "CB_X=0" "CB_TMA_LASTW=1"; do env $env timeout 300 python bench.py --no-breakdown --no-cpu-baseline --no-variants 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('$env',round(d['value']),d['ms_per_step'],d['step_phases_us'])"; done
CB_TMA_LASTW=1 timeout 200 python tools/ktrace.py cfg4 2>&1 | grep -E "acc-ready|epilogue-done"

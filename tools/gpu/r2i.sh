# K7 fixed cost vs batch, skeleton variants, per-tile trace; K0 launch-bounds A/B
set -o pipefail
mkdir -p gpurun_out/r2i
for b in 2 4 8 16 32 64; do echo "== N=$b"; CB_KT_BATCH=$b timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1; done > gpurun_out/r2i/k7_batch.log 2>&1; cat gpurun_out/r2i/k7_batch.log
for env in "CB_TS_DEBUG=28" "CB_TS_DEBUG=29" "CB_TS_DEBUG=20" "CB_TS_DEBUG=12" "CB_TS_NWIN=2" "CB_TS_NWIN=3"; do
  echo "== $env"; env $env timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1
done > gpurun_out/r2i/k7_dbg.log 2>&1; cat gpurun_out/r2i/k7_dbg.log
for b in 2 16; do CB_KT_BATCH=$b CB_TS_DEBUG=28 timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1; done >> gpurun_out/r2i/k7_dbg.log; tail -2 gpurun_out/r2i/k7_dbg.log
timeout 120 python tools/ts_trace.py cfg3 > gpurun_out/r2i/ts_trace.log 2>&1; echo "trace rc=$?"; head -60 gpurun_out/r2i/ts_trace.log
for mb in 1 6; do echo "== CB_K0_MINB=$mb"; CB_K0_MINB=$mb CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg4 2>&1 | tail -1; done > gpurun_out/r2i/k0.log 2>&1; cat gpurun_out/r2i/k0.log
for mb in 1 6 1 6; do CB_K0_MINB=$mb timeout 300 python bench.py --no-breakdown --no-cpu-baseline --no-variants 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().splitlines()[-1]);print('MINB=$mb',d['value'],d['ms_per_step'],d['step_phases_us'])"; done

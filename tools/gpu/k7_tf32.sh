# K7 3xTF32 on cfg3: parity, time (two K halves vs one whole buffer), stage elimination
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs" 2>&1 | tail -2
for rep in 1 2; do
echo "halves:       $(timeout 300 python tools/ktime.py cfg3 tc3xtf32 2>&1 | tail -1)"
echo "whole buffer: $(CB_TS_NO_HALVES=1 timeout 300 python tools/ktime.py cfg3 tc3xtf32 2>&1 | tail -1)"
done
for d in 9 24 8; do echo "halves debug $d: $(CB_TS_DEBUG=$d timeout 300 python tools/ktime.py cfg3 tc3xtf32 2>&1 | tail -1)"; done

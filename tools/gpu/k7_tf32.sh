# K7 3xTF32 on cfg3: parity, time (two K halves vs one whole buffer), stage elimination
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs or model_layers" 2>&1 | tail -2
for rep in 1 2; do
echo "tf32 halves:       $(CB_KT_COLD=1 timeout 300 python tools/ktime.py cfg3 tc3xtf32 2>&1 | tail -1)"
echo "tf32 whole buffer: $(CB_TS_NO_HALVES=1 timeout 300 python tools/ktime.py cfg3 tc3xtf32 2>&1 | tail -1)"
echo "bf16:              $(CB_KT_COLD=1 timeout 300 python tools/ktime.py cfg3 tc3xbf16 2>&1 | tail -1)"
done

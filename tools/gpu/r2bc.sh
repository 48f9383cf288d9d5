# K7 mixed reduction layout (no pad taps): parity + time, producer warps per quadrant 1 / 3, vs padded pairs.
mkdir -p _ab gpurun_out/r2bc
for k in 1 3; do python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=$k',), out='_ab/k$k.so')" > /dev/null 2>&1 || echo fail; done
CB_LIB_PATH=_ab/k1.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs or model_layers or sweep_plan" 2>&1 | tail -2
CB_LIB_PATH=_ab/k3.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs" 2>&1 | tail -2
for rep in 1 2; do for k in 1 3; do for m in 1 2; do
echo "kparts $k pairmode $m: $(CB_TS_PAIRMODE=$m CB_LIB_PATH=_ab/k$k.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done; done; done
for d in 9 24 17; do echo "k1 mixed debug $d: $(CB_TS_DEBUG=$d CB_LIB_PATH=_ab/k1.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done

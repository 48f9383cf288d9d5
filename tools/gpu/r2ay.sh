# K7: producer warps per quadrant x groups per tcgen05.st.
mkdir -p gpurun_out/r2ay _ab
CFGS=("1 1" "1 2" "1 4" "2 2" "2 4" "3 4")
for cfg in "${CFGS[@]}"; do set -- $cfg
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=$1','-DCB_TS_STW=$2'), out='_ab/k$1w$2.so')" > gpurun_out/r2ay/build_k$1w$2.log 2>&1 || echo "build k$1 w$2 failed"
done
for rep in 1 2; do
for cfg in "${CFGS[@]}"; do set -- $cfg
echo "kparts $1 stw $2: $(CB_LIB_PATH=_ab/k$1w$2.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done
done
CB_LIB_PATH=_ab/k1w4.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs" 2>&1 | tail -2

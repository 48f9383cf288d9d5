# K7: window-before-weights order; producer warps per quadrant 2 / 3 / 4 with the pipelined tile loop.
mkdir -p gpurun_out/r2aw _ab
for k in 2 4; do
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=$k',), out='_ab/k$k.so')" > gpurun_out/r2aw/build_k$k.log 2>&1 || echo "build k$k failed"
done
for rep in 1 2; do
timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1
for k in 2 4; do CB_LIB_PATH=_ab/k$k.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1; done
done

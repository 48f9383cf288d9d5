# K7: producer warps per quadrant x load depth.
mkdir -p gpurun_out/r2ax _ab
for cfg in "1 3" "1 5" "2 3" "2 4" "2 6" "3 2"; do set -- $cfg
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=$1','-DCB_TS_DEPTH=$2'), out='_ab/k$1d$2.so')" > gpurun_out/r2ax/build_k$1d$2.log 2>&1 || echo "build k$1 d$2 failed"
done
for rep in 1 2; do
for cfg in "1 3" "1 5" "2 3" "2 4" "2 6" "3 2"; do set -- $cfg
echo "kparts $1 depth $2: $(CB_LIB_PATH=_ab/k$1d$2.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done
done

# K7: which stage paces a tile?  CB_TS_DEBUG bits: 1 no MMA, 16 no A build, 8 no epilogue stores, 4 no input TMA.
mkdir -p _ab
for k in 1 3; do python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=$k',), out='_ab/k$k.so')" > /dev/null 2>&1 || echo fail; done
for k in 1 3; do for d in 0 1 16 8 9 24 17 25 4; do
echo "kparts $k debug $d: $(CB_TS_DEBUG=$d CB_LIB_PATH=_ab/k$k.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done; done

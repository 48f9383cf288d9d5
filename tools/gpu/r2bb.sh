# K7 timing experiment: smaller window TMA boxes (results wrong) -- what would a low-halo 2-D tile buy?
mkdir -p _ab
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=1',), out='_ab/k1.so')" > /dev/null 2>&1 || echo fail
for r in 11 8 4 2; do for d in 0 25 9 24; do
echo "rows $r debug $d: $(CB_TS_HACK_ROWS=$r CB_TS_DEBUG=$d CB_LIB_PATH=_ab/k1.so timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done; done

for rep in 1 2; do for cg in 1 2; do echo "cg $cg: $(CB_TS_CG=$cg timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done; done
for d in 25 9 24 17; do echo "cg2 debug $d: $(CB_TS_CG=2 CB_TS_DEBUG=$d timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done
CB_TS_CG=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs" 2>&1 | tail -2

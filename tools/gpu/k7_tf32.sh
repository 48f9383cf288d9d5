timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few" 2>&1 | tail -6
timeout 300 python tools/ktime.py cfg3 tc3xtf32 2>&1 | tail -2
CB_NO_TS_TF32=1 timeout 300 python tools/ktime.py cfg3 tc3xtf32 2>&1 | tail -1

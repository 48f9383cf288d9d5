for c in cfg1 cfg2b; do CB_TMA_TRACE=1 timeout 600 python tools/ktrace.py $c tc3xbf16 2>&1 | tail -12; done
for c in cfg1 cfg2a cfg2b; do CB_KT_COLD=1 timeout 300 python tools/ktime.py $c tc3xbf16 2>&1 | tail -2; done

for rep in 1 2; do for v in 0 1; do
if [ $v = 1 ]; then export CB_NO_PDL=1; else unset CB_NO_PDL; fi
echo "no_pdl=$v: $(CB_KT_COLD=1 timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done; done
unset CB_NO_PDL
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few or baseline_configs or model_layers or run_single_graph" 2>&1 | tail -2
for nb in 2 8; do echo "N=$nb: $(CB_KT_BATCH=$nb timeout 300 python tools/ktime.py cfg3 2>&1 | tail -1)"; done

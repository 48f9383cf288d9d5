mkdir -p gpurun_out/r2f
K=n1_c256x224x224_f32x7x7_s1x1_p3x3_d1x1_g1_b0
for v in tc3xtf32 tc3xbf16; do for m in main baseline; do echo "== $m $v"; timeout 60 python tools/one_op.py $K $m $v; echo "rc=$?"; done; done > gpurun_out/r2f/hang.log 2>&1
cat gpurun_out/r2f/hang.log
timeout 900 python tools/sweep.py --min-gflop 20 --max-gflop 45 --warmups 1 --runs 2 --out gpurun_out/r2f/sw > gpurun_out/r2f/sw.log 2>&1; echo "sweep20-45 rc=$?"; tail -3 gpurun_out/r2f/sw.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2f/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2f/pytest.log

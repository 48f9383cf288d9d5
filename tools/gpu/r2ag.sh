set -o pipefail
mkdir -p gpurun_out/r2ag
CB_LIB_PATH=_ab/libconvb200_k4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "direct_few" > gpurun_out/r2ag/pytest.log 2>&1; echo "pytest k4 rc=$?"; tail -2 gpurun_out/r2ag/pytest.log
for lib in "" "_ab/libconvb200_k4.so" "" "_ab/libconvb200_k4.so"; do echo "== lib=$lib"; CB_LIB_PATH=$lib CB_KT_COLD=1 timeout 120 python tools/ktime.py cfg3 2>&1 | tail -1; done > gpurun_out/r2ag/k7.log 2>&1; cat gpurun_out/r2ag/k7.log

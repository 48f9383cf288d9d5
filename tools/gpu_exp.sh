set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
timeout 300 python tools/ktime.py pack cfg1 cfg2a cfg2b cfg3 cfg4 2>&1 | tail -10

timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "direct_few" 2>&1 | tail -4

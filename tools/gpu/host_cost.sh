timeout 600 python tools/host_cost.py cfg1 cfg3 2>&1 | tail -12
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1

set -o pipefail
timeout 240 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 200 python tools/phase_probe.py n1_c256x14x14_f256x3x3_s1x1_p1x1_d1x1_g1_b0 2>&1 | tail -3
timeout 200 python tools/devtime.py cfg4 2>&1 | tail -12

# K7 on other few-channel shapes: one producer warp per quadrant (default) vs three.
mkdir -p _ab
python -c "from paper_2407_10730_b200.build import build; build(defines=('-DCB_TS_KPARTS=3',), out='_ab/k3.so')" > /dev/null 2>&1 || echo fail
KEYS="n1_c8x112x112_f64x3x3_s1x1_p1x1_d1x1_g1_b0 n1_c16x112x112_f64x3x3_s1x1_p1x1_d1x1_g1_b0 n1_c16x224x224_f32x3x3_s1x1_p1x1_d1x1_g1_b0 n1_c4x224x224_f64x3x3_s1x1_p1x1_d1x1_g1_b0 n1_c3x224x224_f64x3x3_s1x1_p1x1_d1x1_g1_b0 n1_c3x224x224_f128x5x5_s1x1_p2x2_d1x1_g1_b0 n1_c4x224x224_f256x7x7_s1x1_p3x3_d1x1_g1_b0 n1_c8x224x224_f128x3x3_s2x2_p1x1_d1x1_g1_b0 n1_c16x224x224_f16x1x1_s1x1_p0x0_d1x1_g1_b0 n1_c3x224x224_f16x7x7_s2x2_p3x3_d1x1_g1_b0 n1_c4x112x112_f512x3x3_s2x2_p1x1_d1x1_g1_b0 n16_c3x224x224_f64x7x7_s2x2_p3x3_d1x1_g1_b0"
echo "== kparts 1"; timeout 600 python tools/key_time.py $KEYS 2>&1 | grep us
echo "== kparts 3"; CB_LIB_PATH=_ab/k3.so timeout 600 python tools/key_time.py $KEYS 2>&1 | grep us

# launch list of small single-phase (FFMA) fused ops
mkdir -p gpurun_out/ffma
for key in n1_c128x28x28_f256x3x3_s2x2_p1x1_d1x1_g1_b0 n1_c256x56x56_f64x1x1_s1x1_p0x0_d1x1_g1_b0 n1_c32x14x14_f64x3x3_s1x1_p1x1_d1x1_g1_b0; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/one_op.py $key fused auto 2>/dev/null | grep -v "^==" | python -c "
import sys,csv
rows=list(csv.reader(sys.stdin))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r]
if hi:
    h=rows[hi[0]]; ki=h.index('Kernel Name'); mi=h.index('Metric Value'); gi=h.index('Grid Size')
    for r in rows[hi[0]+1:][-6:]:
        if len(r)>mi: print('   ', r[ki][:60], r[gi], r[mi])
"
echo "== $key"
done

# ncu --set full capture of K7 on cfg3 with source, for per-instruction stall samples.
mkdir -p gpurun_out/k7_ncu
CMD="python tools/ktime.py cfg3"
timeout 300 $CMD > gpurun_out/k7_ncu/plain.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_ts -s 3 -c 1 -o gpurun_out/k7_ncu/k7 -f $CMD > gpurun_out/k7_ncu/ncu.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/k7_ncu

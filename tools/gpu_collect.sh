set -o pipefail
mkdir -p gpurun_out/collect
for c in cfg1 cfg2a cfg2b cfg3 cfg4; do echo "$c $(timeout 60 python tools/ktime.py $c 2>&1 | tail -1)"; done > gpurun_out/collect/ktime.txt
for c in cfg1 cfg2a cfg2b cfg3 cfg4; do echo "$c tf32 $(timeout 60 python tools/ktime.py $c tc3xtf32 2>&1 | tail -1)"; done >> gpurun_out/collect/ktime.txt
timeout 120 python tools/ktime.py pack cfg1 cfg2a cfg2b cfg3 cfg4 > gpurun_out/collect/pack.txt 2>&1
timeout 900 python tools/sweep.py --sample 600 --warmups 3 --runs 10 --device-inputs --out gpurun_out/collect/sweep600 > gpurun_out/collect/sweep.log 2>&1
echo done

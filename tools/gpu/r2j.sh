# stepwise default 3xBF16 (bench table), K8 per-item traces, PCIe probe, K7 full ncu capture
set -o pipefail
mkdir -p gpurun_out/r2j
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2j/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2j/pytest.log
for a in "cfg4 im2col tc3xbf16" "cfg4 sconv tc3xbf16" "cfg4 im2col tc3xtf32" "cfg3 im2col tc3xbf16"; do timeout 120 python tools/k8_trace.py $a 2>&1 | tail -12; done > gpurun_out/r2j/k8_trace.log 2>&1; cat gpurun_out/r2j/k8_trace.log
timeout 120 python tools/h2d_probe.py > gpurun_out/r2j/h2d.log 2>&1; cat gpurun_out/r2j/h2d.log
timeout 900 python bench.py > gpurun_out/r2j/bench.json 2> gpurun_out/r2j/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2j/bench.json').read().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['step_phases_us'], d['e2e']['value'])
for c,row in d['configs'].items():
    print(c, {k:(round(v['operation_us'],1), {p:round(t,1) for p,t in v['phases_us'].items()}) for k,v in row.items()})
print(d['parity']['configs'])
PY
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:conv_ts_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2j/k7_full -f python tools/k7k8_run.py > gpurun_out/r2j/ncu_k7.log 2>&1; echo "ncu rc=$?"

# The real-network op set (configs/model_ops.json: 392 unique layers of 17 torchvision models,
# depthwise / grouped / dilated included) on make_inputs data with CPU-oracle parity on every op.
set -o pipefail
mkdir -p gpurun_out/models
timeout 2400 python tests/sweep_parity.py --opset models --warmups 1 --runs 3 --pending 24 --out gpurun_out/models/models > gpurun_out/models/sweep.log 2>&1; echo "models rc=$?"; tail -30 gpurun_out/models/sweep.log

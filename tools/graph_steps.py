"""Step time of the bench workload with one graph per step vs one graph per ring of steps
(diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs

d = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
RING, STEPS = 4, 48
host = make_inputs(d, RunConfig(seed=0))
dev = [(torch.from_numpy(host.input).cuda(), torch.from_numpy(host.weights).cuda()) for _ in range(RING)]
ys = [torch.empty((d.batch, d.out_channels) + algos.output_shape(d), device="cuda") for _ in range(RING)]
fc = algos.FusedConv(d, "tc3xbf16")
per = [fc.capture(x, w, y) for (x, w), y in zip(dev, ys)]
ring = fc.capture_steps([(x, w, y) for (x, w), y in zip(dev, ys)])


def t(fn, n):
    for i in range(8):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3


for rep in range(3):
    us1 = t(lambda i: per[i % RING].replay(), STEPS) / STEPS
    us4 = t(lambda i: ring.replay(), STEPS // RING) / STEPS
    print(f"per-step graphs {us1:.1f} us/step   ring graph {us4:.1f} us/step")

"""cfg4 e2e step time through HostPipeline for several copy-stream settings (diagnostics)."""
import sys, torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs
d = CONFIGS["cfg4"]
h = make_inputs(d, RunConfig(seed=0))
x = torch.from_numpy(h.input).pin_memory(); w = torch.from_numpy(h.weights).pin_memory()
oh, ow = algos.output_shape(d)
y = torch.empty((d.batch, d.out_channels, oh, ow)).pin_memory()
for hs, ds, depth in ((1, 1, 2), (2, 1, 2), (1, 2, 2), (2, 2, 2), (2, 1, 3), (4, 1, 3)):
    p = algos.HostPipeline(d, copy_streams=hs, d2h_streams=ds, depth=depth)
    for _ in range(5): p.submit(x, w, y)
    p.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); p.wait_streams_for(e0)
    for _ in range(30): p.submit(x, w, y)
    p.record_done(e1); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    print(f"h2d={hs} d2h={ds} depth={depth}: {ms:.3f} ms/step  {algos.flop_count(d) / ms / 1e9:.1f} TFLOP/s", flush=True)

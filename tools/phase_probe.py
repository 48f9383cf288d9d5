"""Per-phase EventLedger times of the drop-ins for a few ops (diagnostics)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import algos, harness
from paper_2407_10730_b200.descriptor import parse_key
from paper_2407_10730_b200.timing import EventLedger, Phase

keys = sys.argv[1:] or ["n1_c4x7x7_f8x1x1_s1x1_p0x0_d1x1_g1_b0", "n1_c64x56x56_f64x3x3_s1x1_p1x1_d1x1_g1_b0"]
for key in keys:
    d = parse_key(key)
    cfg = harness.RunConfig(mode="fused", warmups=3, runs=20)
    inp = harness.device_inputs(d, cfg)
    for name, fn in (("fused", lambda i, l: algos.conv_fused(i, l)),
                     ("baseline", lambda i, l: algos.conv_baseline_im2col_gemm(i, l)),
                     ("main", lambda i, l: algos.conv_main_blocked_direct(i, l))):
        led = EventLedger()
        for _ in range(5):
            led.reset(); fn(inp, led)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = []
        for _ in range(20):
            led.reset(); fn(inp, led); reps.append(led.snapshot())
        host_us = (time.perf_counter() - t0) / 20 * 1e6
        r = reps[-1]
        ph = {p.name: r.elapsed_ns[p] / 1e3 for p in Phase if r.calls[p]}
        print(f"{key[:40]:40s} {name:8s} op={r.operation_ns/1e3:8.1f}us host/call={host_us:7.1f}us "
              + " ".join(f"{k}={v:.1f}" for k, v in ph.items()), flush=True)

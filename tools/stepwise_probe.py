"""Stepwise algorithms' phase times per variant on BASELINE configs (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import os
if os.environ.get("CB_LIB_PATH"):  # A/B runs against another build
    from paper_2407_10730_b200 import _capi as _c
    _c.LIB_PATH = Path(os.environ["CB_LIB_PATH"])
import torch
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device
from paper_2407_10730_b200.timing import EventLedger, Phase, aggregate
for name in sys.argv[1:] or ["cfg4"]:
    d = CONFIGS[name]
    inp = to_device(make_inputs(d, RunConfig(seed=0)))
    for v in ("tc3xtf32", "tc3xbf16"):
        for alg, fn in (("im2col", algos.conv_baseline_im2col_gemm), ("sconv", algos.conv_main_blocked_direct)):
            led = EventLedger(); reps = []
            for r in range(7):
                led.reset(); fn(inp, led, variant=v)
                if r >= 2: reps.append(led.snapshot())
            st = aggregate(reps)
            ph = " ".join(f"{p.name.lower()}={st.phase_ns_mean[p]/1e3:.1f}" for p in Phase if st.calls[p])
            print(f"{name} {v} {alg:7s} op={st.operation_ns_mean/1e3:7.1f}us {ph}", flush=True)

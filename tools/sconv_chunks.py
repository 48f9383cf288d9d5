"""SConv op time vs the chunk budget (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device
from paper_2407_10730_b200.timing import EventLedger, Phase, aggregate
for name in sys.argv[1:] or ["cfg4", "cfg3"]:
    d = CONFIGS[name]
    inp = to_device(make_inputs(d, RunConfig(seed=0)))
    for mb in (126, 252, 504, 2000):
        cache = algos.CacheParams(l2_bytes=mb << 20)
        plan = algos.plan_sconv(d, cache)
        for v in ("tc3xtf32", "tc3xbf16"):
            led = EventLedger(); reps = []
            for r in range(6):
                led.reset(); algos.conv_main_blocked_direct(inp, led, cache, variant=v)
                if r >= 2: reps.append(led.snapshot())
            st = aggregate(reps)
            ph = " ".join(f"{p.name.lower()}={st.phase_ns_mean[p]/1e3:.1f}" for p in Phase if st.calls[p])
            print(f"{name} l2={mb}MB chunks={len(plan.chunks)} {v} op={st.operation_ns_mean/1e3:7.1f}us {ph}", flush=True)

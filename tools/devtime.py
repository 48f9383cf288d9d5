"""Developer timing: CUDA-event time of each kernel path on the BASELINE configs.

    python tools/devtime.py [cfg ...]        (GPU box)
Not the bench (see bench.py); no oracle; prints one line per (config, path).
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from paper_2407_10730_b200 import algos
from paper_2407_10730_b200.configs import CONFIGS, conv_flops, pack_bytes
from paper_2407_10730_b200.timing import EventLedger, Phase


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    return ts[len(ts) // 2] * 1e-3


def main(names):
    p = torch.cuda.get_device_properties(0)
    print(f"# {p.name} sms={p.multi_processor_count} l2={p.L2_cache_size>>20}MB torch={torch.__version__}")
    for name in names:
        d = CONFIGS[name]
        rng = np.random.default_rng(0)
        x = torch.from_numpy((rng.random((d.batch, d.in_channels, d.in_h, d.in_w), dtype=np.float32) * 2 - 1)).cuda()
        w = torch.from_numpy((rng.random((d.out_channels, d.in_channels, d.k_h, d.k_w), dtype=np.float32) * 2 - 1)).cuda()
        inp = algos.ConvInputs(desc=d, input=x, weights=w)
        fl = conv_flops(d)
        for v in ("tc3xtf32", "tc3xbf16", "ffma"):
            packed = algos.pack_fused_weights(w, d, v)
            ws = algos.fused_workspace(d, v) if v != "ffma" else None
            y = torch.empty((d.batch, d.out_channels) + tuple(algos.output_shape(d)), device="cuda")
            t = timeit(lambda: algos.conv_fused(inp, variant=v, packed=packed, workspace=ws, out=y))
            print(f"{name:6s} fused/{v:9s} {t*1e6:9.1f} us  {fl/t/1e12:7.2f} TFLOP/s  "
                  f"layout={algos.fused_layout(d, v) if v != 'ffma' else '-'} plan={algos.fused_plan(d, v)}")
        t = timeit(lambda: algos._im2col_dev(x, d))
        print(f"{name:6s} im2col           {t*1e6:9.1f} us  {pack_bytes(d)/t/1e9:7.1f} GB/s")
        for fn in (algos.conv_baseline_im2col_gemm, algos.conv_main_blocked_direct):
            led = EventLedger()
            for _ in range(3):
                led.reset()
                fn(inp, led)
            rep = led.snapshot()
            parts = " ".join(f"{p.name.lower()}={rep.elapsed_ns[p]/1e3:.1f}us/{rep.calls[p]}"
                             for p in Phase if rep.calls[p])
            print(f"{name:6s} {fn.__name__:28s} op={rep.operation_ns/1e3:9.1f}us {parts}")
        sys.stdout.flush()


def accuracy_vs_k():
    """Normalized max error of each variant against float64 as the reduction grows."""
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    for c, r in [(64, 1), (256, 1), (1024, 1), (256, 3), (1024, 3), (4096, 1), (2048, 7)]:
        d = ConvDescriptor(batch=1, in_channels=c, in_h=14, in_w=14, out_channels=64, k_h=r,
                           k_w=r, pad_h=r // 2, pad_w=r // 2)
        rng = np.random.default_rng(1)
        x = (rng.random((1, c, 14, 14), dtype=np.float32) * 2 - 1)
        w = (rng.random((64, c, r, r), dtype=np.float32) * 2 - 1)
        ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(w).double(),
                                         padding=r // 2).numpy()
        inp = algos.ConvInputs(desc=d, input=x, weights=w)
        errs = {}
        for v in ("tc3xtf32", "tc3xbf16", "ffma"):
            y = algos.conv_fused(inp, variant=v)
            errs[v] = float(np.abs(y.astype(np.float64) - ref).max()) / np.sqrt(c * r * r)
        print(f"acc K={c*r*r:7d} " + " ".join(f"{k}={v:.2e}" for k, v in errs.items()), flush=True)


if __name__ == "__main__":
    if sys.argv[1:2] == ["acc"]:
        accuracy_vs_k()
    else:
        main(sys.argv[1:] or list(CONFIGS))

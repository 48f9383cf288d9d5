"""Per-CTA timeline of one fused-conv (K6) launch from globaltimer stamps (diagnostics).

    CB_TMA_TRACE=1 [CB_TMA_TAIL=0 ...] python tools/ktrace.py cfg4 [variant]
Slots: 0 = epilogue ready, 1..n = accumulator of item k ready (MMAs done), 31 = epilogue
finished.  Times in microseconds relative to the earliest stamp.
"""

from __future__ import annotations

import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
# the timelines exist only in the diagnostics build: point the loader at it before the
# package is imported, then (re)build it if it is missing or stale
os.environ.setdefault("CB_LIB_PATH", str(Path(__file__).resolve().parent.parent / "_ab" / "libconvb200_trace.so"))
from paper_2407_10730_b200.build import trace_lib  # noqa: E402
trace_lib()
os.environ.setdefault("CB_TMA_TRACE", "1")

import numpy as np
import torch

from paper_2407_10730_b200 import _capi, algos
from paper_2407_10730_b200.configs import CONFIGS


def main(name="cfg4", variant="tc3xbf16"):
    d = CONFIGS[name]
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.random((d.batch, d.in_channels, d.in_h, d.in_w), dtype=np.float32) * 2 - 1).cuda()
    w = torch.from_numpy(rng.random((d.out_channels, d.in_channels, d.k_h, d.k_w), dtype=np.float32) * 2 - 1).cuda()
    inp = algos.ConvInputs(desc=d, input=x, weights=w)
    packed = algos.pack_fused_weights(w, d, variant)
    ws = algos.fused_workspace(d, variant)
    for _ in range(3):
        algos.conv_fused(inp, variant=variant, packed=packed, workspace=ws)
    torch.cuda.synchronize()
    lib = _capi.load()
    fn = lib.cb_debug_trace
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    fn.restype = ctypes.c_int
    buf = (ctypes.c_ulonglong * (1024 * 32))()
    slots = ctypes.c_int()
    n = fn(buf, 1024, ctypes.byref(slots))
    a = np.frombuffer(buf, dtype=np.uint64)[: n * slots.value].reshape(n, slots.value).astype(np.float64)
    t0 = a[a > 0].min()
    rel = np.where(a > 0, (a - t0) / 1e3, np.nan)
    print(f"{name} {variant} plan={algos.fused_plan(d, variant)} ctas={n}")
    starts = rel[:, 0]
    ends = rel[:, -1]
    print(f"  epilogue-ready  min {np.nanmin(starts):7.1f} max {np.nanmax(starts):7.1f} us")
    for k in range(1, 13):
        col = rel[:, k]
        if np.all(np.isnan(col)):
            break
        print(f"  item {k - 1} acc-ready min {np.nanmin(col):7.1f} med {np.nanmedian(col):7.1f} "
              f"max {np.nanmax(col):7.1f} us  (ctas {int(np.sum(~np.isnan(col)))})")
    print(f"  epilogue-done   min {np.nanmin(ends):7.1f} med {np.nanmedian(ends):7.1f} max {np.nanmax(ends):7.1f} us")
    for s, label in ((20, "part written"), (21, "part published"), (22, "owner waits"),
                     (23, "owner released"), (24, "partials added")):
        col = rel[:, s]
        if not np.all(np.isnan(col)):
            print(f"  {label:15s} min {np.nanmin(col):7.1f} med {np.nanmedian(col):7.1f} "
                  f"max {np.nanmax(col):7.1f} us  (ctas {int(np.sum(~np.isnan(col)))})")
    order = np.argsort(ends)
    print("  slowest CTAs:", [(int(i), [round(float(v), 1) for v in rel[i, :4]], round(float(ends[i]), 1)) for i in order[-4:]])


if __name__ == "__main__":
    main(*(sys.argv[1:] or []))

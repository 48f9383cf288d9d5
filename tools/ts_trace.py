"""Per-tile timeline of K7 (conv_ts_kernel) from clock64 stamps, CTA 0..3 (diagnostics).

    CB_TS_TRACE=1 python tools/ts_trace.py [cfg3]
Events: 0 TMA issue, 1/2/3/4 producer warp 0: window landed (the barrier test of the NEXT
tile's window passed) / build starts (top of the tile loop) / A written / st drained,
5/6 MMA: A full / accumulator free, 10 commit, 7/8/9 epilogue: accumulator ready / released /
last store issued, 15: kernel start.  (Events 11-14 were a second producer warp of the same
quadrant; with one producer warp per quadrant they are not stamped.)
"""
import ctypes, os, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
# the timelines exist only in the diagnostics build: point the loader at it before the
# package is imported, then (re)build it if it is missing or stale
os.environ.setdefault("CB_LIB_PATH", str(Path(__file__).resolve().parent.parent / "_ab" / "libconvb200_trace.so"))
from paper_2407_10730_b200.build import trace_lib  # noqa: E402
trace_lib()
os.environ.setdefault("CB_TS_TRACE", "1")
import numpy as np
import torch
from paper_2407_10730_b200 import _capi, algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
inp = to_device(make_inputs(CONFIGS[name], RunConfig(seed=0)))
for _ in range(3):
    algos.conv_fused(inp)
torch.cuda.synchronize()
lib = _capi.load()
fn = lib.cb_debug_trace
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
fn.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * (1024 * 32))()
slots = ctypes.c_int()
fn(buf, 1024, ctypes.byref(slots))
a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 16, 512).astype(np.int64)
names = {0: "tma", 1: "p0_sfull", 2: "p0_start", 3: "p0_built", 4: "p0_drained", 5: "mma_afull",
         6: "mma_accfree", 10: "mma_commit", 7: "epi_acc", 8: "epi_release", 9: "epi_stored"}
for cta in range(2):
    t0 = a[cta, 15, 0]
    n = int((a[cta, 7] > 0).sum())
    print(f"CTA {cta}: {n} tiles, kernel start at 0, cycles")
    order = [0, 1, 2, 3, 4, 5, 6, 10, 7, 8, 9]
    print("tile " + " ".join(f"{names[e]:>11s}" for e in order))
    for i in range(n):
        print(f"{i:4d} " + " ".join(f"{a[cta, e, i] - t0:11d}" for e in order))
    d = lambda e1, e0: np.median(a[cta, e1, 2:n] - a[cta, e0, 2:n])
    per_tile = np.median(np.diff(a[cta, 10, :n]))
    print(f"median per tile {per_tile:.0f}; p0 build {d(3,2):.0f} drain {d(4,3):.0f}; "
          f"mma wait acc {d(6,5):.0f}; commit-issue {d(10,6):.0f}; epi acc->release {d(8,7):.0f} ->stored {d(9,7):.0f}")

"""Per-item timeline of K8 (gemm_ts_kernel) from globaltimer stamps (diagnostics).

    python tools/k8_trace.py [cfg4] [im2col|sconv] [tc3xbf16|tc3xtf32]
Stamps (CB_K8_TRACE): per local item li < 5 of every CTA, producer warp 0 start / end, MMA
first chunk / last commit, epilogue accumulator ready / last store; kernel start / end.
"""
import ctypes, os, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
# the timelines exist only in the diagnostics build: point the loader at it before the
# package is imported, then (re)build it if it is missing or stale
os.environ.setdefault("CB_LIB_PATH", str(Path(__file__).resolve().parent.parent / "_ab" / "libconvb200_trace.so"))
from paper_2407_10730_b200.build import trace_lib  # noqa: E402
trace_lib()
os.environ["CB_K8_TRACE"] = "1"
import numpy as np
import torch
from paper_2407_10730_b200 import _capi, algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device
from paper_2407_10730_b200.timing import PhaseLedger

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
path = sys.argv[2] if len(sys.argv) > 2 else "im2col"
variant = sys.argv[3] if len(sys.argv) > 3 else "tc3xbf16"
inp = to_device(make_inputs(CONFIGS[name], RunConfig(seed=0)))
fn = algos.conv_baseline_im2col_gemm if path == "im2col" else algos.conv_main_blocked_direct
for _ in range(3):
    fn(inp, PhaseLedger(), variant=variant)
torch.cuda.synchronize()
lib = _capi.load()
f = lib.cb_debug_trace
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
f.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * (1024 * 32))()
slots = ctypes.c_int()
n = f(buf, 1024, ctypes.byref(slots))
full = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
a = full.reshape(1024, 32)[:256]
n = int((a[:, 31] > 0).sum())
a = a[:n]
ch = full[8192:8192 + 4 * 256].reshape(256, 4)
t0 = a[:, 31][a[:, 31] > 0].min()
rel = lambda v: np.where(v > 0, v - t0, -1)
start, end = rel(a[:, 31]), rel(a[:, 30])
print(f"{name} {path} {variant}: {n} CTAs; start spread {start.min()}..{start.max()} ns; "
      f"end min/median/max {end.min()}/{int(np.median(end))}/{end.max()} ns")
items = [(a[:, li * 6 + 2] > 0).sum() for li in range(5)]
print("CTAs with local item li:", items)
ev = ["p_start", "p_end", "mma_first", "mma_commit", "epi_ready", "epi_done"]
for li in range(5):
    if items[li] == 0:
        break
    m = a[:, li * 6 + 2] > 0
    cols = {e: rel(a[m, li * 6 + k]) for k, e in enumerate(ev)}
    med = {e: int(np.median(v)) for e, v in cols.items()}
    print(f"item {li}: median " + " ".join(f"{e}={v}" for e, v in med.items()) +
          f" | mma {int(np.median(cols['mma_commit'] - cols['mma_first']))} ns"
          f" epi {int(np.median(cols['epi_done'] - cols['epi_ready']))} ns"
          f" | max epi_done {cols['epi_done'].max()}")
for c in (0, 1, n // 2, n - 1):
    print(f"CTA {c}: start {start[c]} end {end[c]} | " + " ; ".join(
        ",".join(str(rel(a[c, li * 6 + k])) for k in range(6)) for li in range(5) if a[c, li * 6 + 2] > 0))

nc = int((ch[:, 3] > 0).sum())
print(f"CTA 0 chunks ({nc}): tma_issue, prod_saw_stage, prod_a_full, mma_saw_a_full (ns from start)")
for c in list(range(min(nc, 12))) + list(range(max(12, nc - 6), nc)):
    print(f"  {c:3d} " + " ".join(f"{rel(ch[c, e]):8d}" for e in range(4)))
if nc > 8:
    d = np.diff(ch[:nc, 3])
    lat = ch[:nc, 1] - ch[:nc, 0]
    print(f"  per-chunk MMA pace median {int(np.median(d))} ns; TMA issue -> producer sees stage median "
          f"{int(np.median(lat))} ns; producer stage -> a_full {int(np.median(ch[:nc, 2] - ch[:nc, 1]))} ns; "
          f"a_full -> MMA {int(np.median(ch[:nc, 3] - ch[:nc, 2]))} ns")

"""Host-side cost per C-ABI call (diagnostics): N back-to-back calls, host clock."""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import _capi, algos, harness
from paper_2407_10730_b200.descriptor import parse_key
from paper_2407_10730_b200.timing import EventLedger, Phase

key = sys.argv[1] if len(sys.argv) > 1 else "n1_c64x56x56_f64x3x3_s1x1_p1x1_d1x1_g1_b0"
d = parse_key(key)
inp = harness.device_inputs(d, harness.RunConfig())
lib = _capi.load()
v = "tc3xbf16"
pr = algos._prep(d, v)
lay = algos.fused_layout(d, v)
ws = torch.empty(lay["workspace_bytes"], dtype=torch.uint8, device="cuda")
hi, lo, _ = algos.pack_fused_weights(inp.weights, d, v)
y = torch.empty((1, d.out_channels, pr.oh, pr.ow), device="cuda")
st = torch.cuda.current_stream().cuda_stream
x = inp.input
calls = {
    "pack_weights": lambda: lib.cb_fused_pack_weights(pr.vid, pr.pcd, inp.weights.data_ptr(), hi.data_ptr(), lo.data_ptr(), st),
    "pack_input": lambda: lib.cb_fused_pack_input(pr.vid, pr.pcd, x.data_ptr(), ws.data_ptr(), ws.numel(), st),
    "conv_fused_packed": lambda: lib.cb_conv_fused_packed(pr.vid, pr.pcd, x.data_ptr(), ws.data_ptr(), ws.numel(), hi.data_ptr(), lo.data_ptr(), None, None, y.data_ptr(), st),
    "output_shape": lambda: lib.cb_version(),
}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for name, fn in calls.items():
    for _ in range(20): fn()
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:20s} host {1e6 * (t1 - t0) / n:7.2f} us/call", flush=True)
t0 = time.perf_counter()
for _ in range(1000): ev[0].record()
print(f"event.record        host {1e6 * (time.perf_counter() - t0) / 1000:7.2f} us/call")
t0 = time.perf_counter()
for _ in range(1000): torch.cuda.current_stream()
print(f"current_stream      host {1e6 * (time.perf_counter() - t0) / 1000:7.2f} us/call")
led = EventLedger()
t0 = time.perf_counter()
for _ in range(200):
    led.reset(); led.start(Phase.IN_PACKING); led.update(Phase.IN_PACKING)
print(f"ledger start+update host {1e6 * (time.perf_counter() - t0) / 200:7.2f} us/pair")
# device: kernel alone, back to back
for name in ("pack_input", "conv_fused_packed"):
    fn = calls[name]
    torch.cuda.synchronize(); ev[0].record()
    for _ in range(100): fn()
    ev[1].record(); torch.cuda.synchronize()
    print(f"{name:20s} device {ev[0].elapsed_time(ev[1]) * 10:7.2f} us/launch (back to back)")
# host-only entry points
fl = _capi.CbFusedLayout(); tp = _capi.CbTilePlan()
oh, ow = ctypes.c_int(), ctypes.c_int()
host_only = {
    "fused_layout_query": lambda: lib.cb_fused_layout_query(pr.vid, pr.pcd, ctypes.byref(fl)),
    "fused_plan_tiles": lambda: lib.cb_fused_plan_tiles(pr.vid, pr.pcd, ctypes.byref(tp)),
    "output_shape": lambda: lib.cb_output_shape(pr.pcd, ctypes.byref(oh), ctypes.byref(ow)),
    "conv_fused_packed(ws too small)": lambda: lib.cb_conv_fused_packed(pr.vid, pr.pcd, x.data_ptr(), ws.data_ptr(), 16, hi.data_ptr(), lo.data_ptr(), None, None, y.data_ptr(), st),
}
for name, fn in host_only.items():
    for _ in range(20): fn()
    t0 = time.perf_counter()
    for _ in range(2000): fn()
    print(f"{name:32s} host {1e6 * (time.perf_counter() - t0) / 2000:7.2f} us/call", flush=True)
import os
print("environ size", len(os.environ))

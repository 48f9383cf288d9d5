"""Host-side cost of one launch call of each fused-path entry point (diagnostics): the time the
C ABI call takes to return, averaged over back-to-back asynchronous calls.

    python tools/host_cost.py [cfg1 cfg3 ...]
"""
import ctypes
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2407_10730_b200 import _capi, algos
from paper_2407_10730_b200.configs import CONFIGS
from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device

lib = _capi.load()
for name in sys.argv[1:] or ["cfg1", "cfg2b", "cfg3"]:
    d = CONFIGS[name]
    inp = to_device(make_inputs(d, RunConfig(seed=0)))
    for variant in ("tc3xbf16", "ffma"):
        cd, vid = _capi.cdesc(d), _capi.variant_id(variant)
        hi, lo, wf = algos.pack_fused_weights(inp.weights, d, variant)
        ws = algos.fused_workspace(d, variant)
        nbytes = ws.numel() if ws is not None else 0
        wsp = ws.data_ptr() if ws is not None else None
        y = torch.empty((d.batch, d.out_channels) + algos.output_shape(d), device="cuda")
        ptr = lambda t: None if t is None else t.data_ptr()
        st = torch.cuda.current_stream().cuda_stream
        calls = {"K6/K7 cb_conv_fused_packed": lambda: lib.cb_conv_fused_packed(
            vid, ctypes.byref(cd), inp.input.data_ptr(), wsp, nbytes, ptr(hi), ptr(lo), ptr(wf), None,
            y.data_ptr(), st)}
        if variant != "ffma":
            calls["K0 cb_fused_pack_input"] = lambda: lib.cb_fused_pack_input(
                vid, ctypes.byref(cd), inp.input.data_ptr(), wsp, nbytes, st)
            calls["K3 cb_fused_pack_weights"] = lambda: lib.cb_fused_pack_weights(
                vid, ctypes.byref(cd), inp.weights.data_ptr(), ptr(hi), ptr(lo), st)
        for label, fn in calls.items():
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            n = 200
            t0 = time.perf_counter()
            for _ in range(n):
                fn()
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            print(f"{name} {variant:9s} {label:28s} host {1e6 * (t1 - t0) / n:6.1f} us/call, "
                  f"device-bound total {1e6 * (t2 - t0) / n:6.1f} us/call", flush=True)
        t0 = time.perf_counter()
        for _ in range(200):
            algos.conv_fused(inp, variant=variant)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{name} {variant:9s} {'algos.conv_fused (whole op)':28s} host {1e6 * (t1 - t0) / 200:6.1f} us/call", flush=True)

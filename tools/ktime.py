"""Kernel-only timing of the fused conv (K6) and its packing kernels, back to back.

    CB_TMA_CG=2 CB_TMA_BN=256 CB_TMA_DEBUG=0 python tools/ktime.py cfg4 [variant]
Launches are enqueued back to back between two CUDA events, so host overhead is hidden
whenever a launch takes longer than its host-side call.  Diagnostics only.
"""

from __future__ import annotations

import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from bench import Clocks
from paper_2407_10730_b200 import _capi, algos
from paper_2407_10730_b200.configs import CONFIGS, conv_flops


_FLUSH = []


def cold_time(fn, reps: int) -> float:
    """us per launch of fn with the L2 flushed before each launch (a 256 MB write, then a
    256 MB read so the flush lines are clean): one graph of reps x (flush, fn) minus one
    graph of reps x flush."""
    if not _FLUSH:
        _FLUSH.extend([torch.empty(64 << 20, device="cuda"), torch.ones(64 << 20, device="cuda")])
    fw, fr = _FLUSH

    def flush():
        fw.zero_()
        fr.sum()
    out = []
    for with_fn in (True, False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                flush()
                if with_fn:
                    fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / reps * 1e3)
    return out[0] - out[1]


def run(name: str, variant: str, reps: int = 20) -> None:
    d = CONFIGS[name]
    if os.environ.get("CB_KT_BATCH"):  # diagnostics: same layer, another batch size
        from dataclasses import replace
        d = replace(d, batch=int(os.environ["CB_KT_BATCH"]))
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.random((d.batch, d.in_channels, d.in_h, d.in_w), dtype=np.float32) * 2 - 1).cuda()
    w = torch.from_numpy(rng.random((d.out_channels, d.in_channels, d.k_h, d.k_w), dtype=np.float32) * 2 - 1).cuda()
    y = torch.empty((d.batch, d.out_channels) + algos.output_shape(d), device="cuda")
    lib = _capi.load()
    cd = _capi.cdesc(d)
    vid = _capi.variant_id(variant)
    hi, lo, wf = algos.pack_fused_weights(w, d, variant)
    ws = algos.fused_workspace(d, variant)
    nbytes = ws.numel() if ws is not None else 0
    wsp = ws.data_ptr() if ws is not None else None
    cur = lambda: torch.cuda.current_stream().cuda_stream  # graph capture uses its own stream
    ptr = lambda t: None if t is None else t.data_ptr()

    def k0():
        _capi.check(lib.cb_fused_pack_input(vid, ctypes.byref(cd), x.data_ptr(), wsp, nbytes, cur()))

    def k6():
        _capi.check(lib.cb_conv_fused_packed(vid, ctypes.byref(cd), x.data_ptr(), wsp, nbytes,
                                             ptr(hi), ptr(lo), ptr(wf), None, y.data_ptr(), cur()))

    def k3():
        _capi.check(lib.cb_fused_pack_weights(vid, ctypes.byref(cd), w.data_ptr(), ptr(hi),
                                              ptr(lo), cur()))

    k0()
    res = {}
    clk = None
    for label, fn in (("K3", k3), ("K0", k0), ("K6", k6)):
        if fn is not k6 and variant == "ffma":
            continue
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        # device time: the reps launches replay from one CUDA graph (no host gaps)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(reps):
                fn()
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = Clocks(0) if label == "K6" else None
        if sampler:
            sampler.__enter__()
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        if sampler:
            sampler.__exit__(None, None, None)
            clk = sampler.summary()
        res[label] = e0.elapsed_time(e1) / reps * 1e3
        if os.environ.get("CB_KT_COLD"):  # L2-cold: T(flush + launch) - T(flush), per launch
            res[label + "cold"] = cold_time(fn, reps)
    if clk:
        print(f"   clocks during K6: {clk}")
    t6 = res["K6"] * 1e-6
    env = {k: v for k, v in os.environ.items() if k.startswith("CB_")}
    print(f"{name} {variant} env={env} plan={algos.fused_plan(d, variant)}")
    print("   " + " ".join(f"{k}={v:.1f}us" for k, v in res.items()) +
          f"  K6 {conv_flops(d) / t6 / 1e12:.1f} TFLOP/s", flush=True)


if __name__ == "__main__" and (len(sys.argv) < 2 or sys.argv[1] not in ("pack", "ceiling")):
    run(sys.argv[1] if len(sys.argv) > 1 else "cfg4", sys.argv[2] if len(sys.argv) > 2 else "tc3xbf16")


def pack(name: str, reps: int = 20) -> None:
    """K1 (im2col) and K2 (slice pack over all slices) back to back, with GB/s of the
    algorithmic pack bytes."""
    from paper_2407_10730_b200.configs import pack_bytes
    d = CONFIGS[name]
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.random((d.batch, d.in_channels, d.in_h, d.in_w), dtype=np.float32)).cuda()
    lib = _capi.load()
    cd = _capi.cdesc(d)
    oh, ow = algos.output_shape(d)
    kdim = d.in_channels * d.k_h * d.k_w
    cols = torch.empty(kdim * d.batch * oh * ow, device="cuda")
    sp = _capi.CbSlicePlan()
    _capi.check(lib.cb_sconv_plan(ctypes.byref(cd), oh * ow, ctypes.byref(sp)))
    st = torch.cuda.current_stream().cuda_stream
    fns = {"K1 im2col": lambda: _capi.check(lib.cb_im2col_f32(ctypes.byref(cd), x.data_ptr(), cols.data_ptr(), st)),
           "K2 slices": lambda: _capi.check(lib.cb_sconv_pack_f32(ctypes.byref(cd), ctypes.byref(sp), 0, sp.num_slices,
                                                                  x.data_ptr(), cols.data_ptr(), st))}
    for label, fn in fns.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e-3
        print(f"{name} {label}: {t * 1e6:8.1f} us  {pack_bytes(d) / t / 1e9:7.0f} GB/s", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "pack":
    for c in sys.argv[2:] or list(CONFIGS):
        pack(c)


def write_ceiling(nbytes: int = 231 << 20, reps: int = 20) -> None:
    """Plain streaming-write and copy bandwidth on a buffer the size of cfg4's im2col."""
    a = torch.empty(nbytes // 4, device="cuda")
    b = torch.empty_like(a)
    for label, fn, mult in (("fill", lambda: a.fill_(1.0), 1), ("copy", lambda: b.copy_(a), 2)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e-3
        print(f"{label} {nbytes >> 20} MB: {t * 1e6:.1f} us  {mult * nbytes / t / 1e9:.0f} GB/s", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ceiling":
    write_ceiling()

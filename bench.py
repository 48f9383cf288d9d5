#!/usr/bin/env python
"""bench.py -- the B200 conv path on BASELINE.json's headline workload (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--variant tc3xbf16|tc3xtf32|ffma] [--config cfg4] [--scaling weak|strong]

A step is one pass of the path over one batch: the fused implicit-GEMM conv of config 4
(N=128, C=256, 14x14, K=256, 3x3, stride 1, pad 1) through the public
API paper_2407_10730_b200.conv_fused: K3 weight split (PRE_REORDER) + K0 activation
split (IN_PACKING) + K6 tcgen05 conv (IN_MICROKERNEL).  Data is seeded synthetic U(-1,1)
exactly as the reference's make_inputs draws it.

* value        device-resident throughput, GFLOP/s summed over ranks (inputs resident in
               HBM; 4 rotating input/workspace/output sets, 308 MB > 2x L2, so no step
               reuses another's cache lines).  Time = max over ranks of the CUDA-event
               time of exactly K steps between barrier + synchronize.
* e2e          same metric through the same call with pinned HOST buffers: every step
               copies x and w host->device and y device->host inside the timed region.
* roofline     dominant kernel (conv_tma_kernel): algorithmic FLOPs / its mean launch
               time (EventLedger IN_MICROKERNEL), vs the measured dense bf16 peak.
* cpu_baseline the reference's own CPU algorithm (oracle/reference_port.py, a restatement
               of algos.py) on a bounded sample of the same workload, rank 0 at N=1 only.
* breakdown    per-step (phase) CUDA-event times of the three GPU algorithms on the
               workload: Im2col-GEMM, SConv (blocked direct) and fused.

--impl reference: rank 0 times the reference CPU algorithm (port) with all host threads
on the same config/metric and prints the same JSON line with "impl": "reference"; other
ranks exit 0 without work.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"] \
    if (ROOT / "BASELINE.json").exists() else \
    "conv GFLOP/s (2*N*K*P*Q*C*R*S/t) + pack/compute breakdown; % of roofline"
UNIT = "GFLOP/s"
RING = 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-breakdown", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    return rank, world, local


def workload(cfg_name: str, world: int, scaling: str, rank: int):
    from paper_2407_10730_b200.configs import CONFIGS
    d = CONFIGS[cfg_name]
    if scaling == "strong" and world > 1:
        per = d.batch // world + (1 if rank < d.batch % world else 0)
        d = replace(d, batch=max(1, per))
    return d


# ------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return None
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9
                          for i, v in enumerate(r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
# CPU reference (the oracle port of the reference algorithms)
# ------------------------------------------------------------------------------------------
def cpu_reference(d_full, seconds: float, threads: int | None = None, algo: str = "main"):
    """GFLOP/s of the reference CPU algorithm on a bounded sample of the workload:
    batches of `sample_n` images of the same conv until `seconds` have elapsed."""
    import numpy as np
    from oracle import conv_oracle as orc
    from oracle import reference_port as rp
    from paper_2407_10730_b200.descriptor import flop_count
    threads = threads or os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(threads)
    except ImportError:  # pragma: no cover
        limiter = None
    d1 = replace(d_full, batch=min(d_full.batch, 2))
    x, w, b = orc.make_inputs(d1, 0)
    fn = rp.conv_main_blocked_direct if algo == "main" else rp.conv_baseline_im2col_gemm
    done = 0
    t0 = time.perf_counter()
    while True:
        fn(d1, x, w, b)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds or done >= 1000:
            break
    if limiter is not None:
        limiter.unregister() if hasattr(limiter, "unregister") else None
    flops = flop_count(d1) * done
    return {"value": flops / el / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
            "algorithm": f"reference {'conv_main_blocked_direct' if algo == 'main' else 'conv_baseline_im2col_gemm'} "
                         "(oracle/reference_port.py)",
            "sample": f"{done} x {d1.batch} image(s) of the workload conv ({el:.1f} s)",
            "seconds": el}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    d = workload(args.config, 1, "weak", 0)
    from paper_2407_10730_b200.configs import conv_flops
    per_step = max(1.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(args.warmup):
        cpu_reference(d, 0.0)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_reference(d, per_step))
    el = time.perf_counter() - t0
    value = statistics.mean(v["value"] for v in vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U(-1,1), reference make_inputs)",
            "config": {"workload": f"{args.config}: {d}", "global_batch": d.batch,
                       "sample_per_step": vals[0]["sample"]},
            "cpu_baseline": {k: vals[0][k] for k in ("kind", "cores", "sample", "algorithm")} | {"value": value, "unit": UNIT},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    from paper_2407_10730_b200 import _capi, algos
    from paper_2407_10730_b200.configs import conv_flops
    from paper_2407_10730_b200.harness import RunConfig, make_inputs
    from paper_2407_10730_b200.roofline import conv_roofline, load_peaks
    from paper_2407_10730_b200.timing import EventLedger, Phase

    rank, world, local = dist_env()
    variant = args.variant or algos.FUSED_DEFAULT_VARIANT
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _capi.load()
    d = workload(args.config, world, args.scaling, rank)
    flops = conv_flops(d)

    host = make_inputs(d, RunConfig(seed=rank))
    x_h, w_h = host.input, host.weights
    dev = [(torch.from_numpy(x_h).cuda(), torch.from_numpy(w_h).cuda()) for _ in range(RING)]
    ys = [torch.empty((d.batch, d.out_channels) + algos.output_shape(d), device="cuda")
          for _ in range(RING)]
    wss = [algos.fused_workspace(d, variant) for _ in range(RING)] if variant != "ffma" else [None] * RING
    inps = [algos.ConvInputs(desc=d, input=x, weights=w) for x, w in dev]

    def step(i, ledger):
        k = i % RING
        algos.conv_fused(inps[k], ledger, variant=variant, workspace=wss[k], out=ys[k])

    def barrier():
        if dist is not None:
            dist.barrier()

    led = EventLedger()
    for i in range(args.warmup):
        led.reset()
        step(i, led)
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps ----
    reports = []
    ledgers = [EventLedger() for _ in range(args.steps)]
    launches0 = lib.cb_launch_count()
    barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for i in range(args.steps):
            step(i, ledgers[i])
        t1.record()
        torch.cuda.synchronize()
    barrier()
    launches = lib.cb_launch_count() - launches0
    ms = t0.elapsed_time(t1) / args.steps
    reports = [l.snapshot() for l in ledgers]
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tot = torch.tensor([float(flops)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tot)
        total_flops = float(tot.item())
    else:
        total_flops = float(flops)
    value = total_flops / (ms * 1e-3) / 1e9

    kern_ns = statistics.mean(r.elapsed_ns[Phase.IN_MICROKERNEL] for r in reports)
    pack_ns = statistics.mean(r.elapsed_ns[Phase.IN_PACKING] for r in reports)
    wsplit_ns = statistics.mean(r.elapsed_ns[Phase.PRE_REORDER] for r in reports)

    # ---- e2e through the same public call with pinned host buffers ----
    x_p = torch.from_numpy(x_h).pin_memory()
    w_p = torch.from_numpy(w_h).pin_memory()
    y_p = torch.empty(ys[0].shape, dtype=torch.float32).pin_memory()
    inp_h = algos.ConvInputs(desc=d, input=x_p, weights=w_p)
    for _ in range(max(1, args.warmup)):
        algos.conv_fused(inp_h, variant=variant, workspace=wss[0], out=y_p)
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        algos.conv_fused(inp_h, variant=variant, workspace=wss[0], out=y_p)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": total_flops / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": int(x_h.nbytes + w_h.nbytes),
           "d2h_bytes_per_step": int(y_p.numel() * 4)}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    peaks = load_peaks()
    rl = conv_roofline(d, variant, peaks)
    achieved = flops / (kern_ns * 1e-9) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"{args.config}/{variant}", {}).get("dram_bytes")
        except (ValueError, OSError):
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["bf16_tflops"], "traffic": traffic,
                "kernel": "conv_tma_kernel (K6)", "kernel_us": kern_ns / 1e3,
                "peak_source": f"{peaks['source']} dense bf16 (burst)",
                "split_effective_peak": rl["effective_peak_tflops"],
                "frac_of_split_peak": achieved / rl["effective_peak_tflops"],
                "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": rl["bytes"],
                "roofline_us": rl["t_roofline_s"] * 1e6}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.scaling == "weak" else "strong", "vs_baseline": None,
            "dtype": "f32", "compute": f"{variant}: tcgen05 split products, fp32 accumulate in TMEM"
            if variant != "ffma" else "ffma fp32",
            "data": "synthetic (seeded U(-1,1), reference make_inputs)",
            "config": {"workload": f"{args.config}: N={d.batch} C={d.in_channels} {d.in_h}x{d.in_w} "
                                   f"K={d.out_channels} {d.k_h}x{d.k_w} s{d.stride_h} p{d.pad_h}, "
                                   "fused implicit-GEMM conv per step",
                       "global_batch": d.batch * (world if args.scaling == "weak" else 1),
                       "per_gpu_batch": d.batch, "variant": variant,
                       "l2": f"{RING} rotating input/workspace/output sets (> 2x L2); no flush",
                       "parallelism": f"batch-sharded x{world}, no collective on the data path"},
            "gpu_launches": int(launches),
            "launches_per_step": launches / args.steps,
            "step_phases_us": {"pre_reorder(K3 weight split)": wsplit_ns / 1e3,
                               "in_packing(K0 act split)": pack_ns / 1e3,
                               "in_microkernel(K6 conv)": kern_ns / 1e3},
            "roofline": roofline, "e2e": e2e, "clocks": clk.summary()}

    if not args.no_breakdown:
        line["breakdown"] = breakdown(d, variant)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(d, args.cpu_seconds)
        line["cpu_baseline"].pop("seconds", None)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def breakdown(d, fused_variant, runs: int = 5):
    """Per-phase CUDA-event times (us, mean of `runs`) of the three GPU algorithms."""
    import torch
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device
    from paper_2407_10730_b200.timing import EventLedger, Phase, aggregate
    inp = to_device(make_inputs(d, RunConfig(seed=0)))
    out = {}
    for name, fn in (("im2col_gemm", lambda i, l: algos.conv_baseline_im2col_gemm(i, l)),
                     ("sconv", lambda i, l: algos.conv_main_blocked_direct(i, l)),
                     ("fused", lambda i, l: algos.conv_fused(i, l, variant=fused_variant))):
        led = EventLedger()
        reps = []
        for r in range(runs + 2):
            led.reset()
            fn(inp, led)
            if r >= 2:
                reps.append(led.snapshot())
        st = aggregate(reps)
        op = st.operation_ns_mean
        pack = st.phase_ns_mean[Phase.IN_PACKING] + (st.phase_ns_mean[Phase.PRE_REORDER]
                                                    if name == "im2col_gemm" else 0.0)
        out[name] = {"operation_us": op / 1e3,
                     "gflops": algos.flop_count(d) / (op * 1e-9) / 1e9 if op else None,
                     "pack_share": pack / op if op else None,
                     "phases_us": {p.name.lower(): st.phase_ns_mean[p] / 1e3 for p in Phase
                                   if st.calls[p]},
                     "calls": {p.name.lower(): st.calls[p] for p in Phase if st.calls[p]}}
    torch.cuda.synchronize()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

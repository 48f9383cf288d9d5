#!/usr/bin/env python
"""bench.py -- the B200 conv path on BASELINE.json's headline workload (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--variant tc3xbf16|tc3xtf32|ffma] [--config cfg4] [--scaling weak|strong]

A step is one pass of the path over one batch: the fused implicit-GEMM conv of config 4
(N=128, C=256, 14x14, K=256, 3x3, stride 1, pad 1): K3 weight split
(PRE_REORDER) + K0 activation split (IN_PACKING) + K6 tcgen05 conv (IN_MICROKERNEL), all
three every step.  Data is seeded synthetic U(-1,1) exactly as the reference's
make_inputs draws it.

* value        device-resident throughput, GFLOP/s summed over ranks: one FusedConv plan,
               one CUDA graph per ring of 4 whole steps (a remainder of K replays per-step
               graphs); 4 rotating input /
               output sets (x 25.7 MB + y 25.7 MB each, plus the 44.6 MB workspace the
               step rewrites: > 2x the 126 MB L2 over a ring cycle).  Time = max over ranks
               of the CUDA-event time of exactly K steps between barrier + synchronize.
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
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
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
    """Samples SM clock and throttle reasons through NVML in a background thread (about
    every 0.5 ms) while the timed region runs; falls back to one nvidia-smi query."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception:  # no NVML: summary() falls back to nvidia-smi
            self._nvml = None
        return self

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((mhz, rs))
            except Exception:
                break
            time.sleep(0.0005)

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self._thread.join(timeout=1)
        return False

    def summary(self):
        if self.samples:
            sm = [s[0] for s in self.samples]
            reasons = sorted({name for _, rs in self.samples for bit, name in self.REASONS.items()
                              if rs & bit})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=10).stdout.strip().split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]), "reasons": [],
                    "samples": 1, "source": "nvidia-smi after the timed region"}
        except Exception:
            return None


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
    variant = algos.resolve_variant(workload(args.config, world, args.scaling, rank),
                                    args.variant or algos.FUSED_AUTO)
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
    # One plan (layout, packed weights, workspace) and one CUDA graph per ring slot; each
    # graph is a full step: K3 weight split + K0 activation split + K6 conv.
    fc = algos.FusedConv(d, variant)
    launches0 = lib.cb_launch_count()
    fc.run(dev[0][0], ys[0], weights=dev[0][1])
    launches_per_step = lib.cb_launch_count() - launches0
    graphs = [fc.capture(x, w, y) for (x, w), y in zip(dev, ys)]
    # the timed stream replays one graph per ring of RING steps (no launch gap between the
    # steps of a ring); a remainder of steps replays the per-step graphs
    ring_graph = fc.capture_steps([(x, w, y) for (x, w), y in zip(dev, ys)])

    def run_steps(k: int) -> None:
        for _ in range(k // RING):
            ring_graph.replay()
        for i in range(k % RING):
            graphs[i].replay()
    # Instrumented copies of the same step graphs: external CUDA events captured between
    # K3 / K0 / K6 re-record on every replay.  Event nodes add launch gaps, so these are
    # replayed in a second pass after the timed region, only to time the kernels.
    slot_ledgers = [EventLedger(external=True) for _ in range(RING)]
    igraphs = [fc.capture(x, w, y, ledger=led) for (x, w), y, led in zip(dev, ys, slot_ledgers)]

    def barrier():
        if dist is not None:
            dist.barrier()

    run_steps(args.warmup)
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps ----
    barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        run_steps(args.steps)
        t1.record()
        torch.cuda.synchronize()
    barrier()
    launches = launches_per_step * args.steps
    ms = t0.elapsed_time(t1) / args.steps

    # per-kernel durations: replay the instrumented graphs as many steps as were timed and
    # read every slot's in-graph events after each ring cycle
    reports = []
    for i in range(max(args.steps, RING)):
        igraphs[i % RING].replay()
        if i % RING == RING - 1:
            reports.extend(led.snapshot() for led in slot_ledgers)
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
    # HostPipeline: the package's host-buffer API -- per step, x and w go host->device and
    # y device->host, on their own streams, overlapping the neighbouring steps' kernels
    pipe = algos.HostPipeline(d, variant)
    for _ in range(max(1, args.warmup)):
        pipe.submit(x_p, w_p, y_p)
    pipe.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    pipe.wait_streams_for(e0)
    for _ in range(args.steps):
        pipe.submit(x_p, w_p, y_p)
    pipe.record_done(e1)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": total_flops / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e2e_ms,
           "api": "HostPipeline.submit (pinned host x, w in; y out; copies overlap kernels)",
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
                       "graph": f"one CUDA graph per {RING} whole steps (K3 + K0 + K6 each)",
                       "parallelism": f"batch-sharded x{world}, no collective on the data path"},
            "gpu_launches": int(launches),
            "launches_per_step": launches / args.steps,
            "step_phases_us": {"pre_reorder(K3 weight split)": wsplit_ns / 1e3,
                               "in_packing(K0 act split)": pack_ns / 1e3,
                               "in_microkernel(K6 conv)": kern_ns / 1e3,
                               "timing": "CUDA events captured in the step graphs, replayed "
                                         f"{len(reports)} steps after the timed region"},
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
    """Per-phase CUDA-event times (us, mean of `runs`) of the three GPU algorithms.  Each
    algorithm is captured once into a CUDA graph with external phase events and replayed
    (the harness's graph mode), so a phase's time is its kernels', not the host's launch
    latency between an eager event and the kernel after it."""
    import torch
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.harness import RunConfig, make_inputs, to_device
    from paper_2407_10730_b200.timing import EventLedger, Phase, aggregate
    inp = to_device(make_inputs(d, RunConfig(seed=0)))
    out = {}
    for name, fn in (("im2col_gemm", lambda i, l: algos.conv_baseline_im2col_gemm(i, l)),
                     ("sconv", lambda i, l: algos.conv_main_blocked_direct(i, l)),
                     ("fused", lambda i, l: algos.conv_fused(i, l, variant=fused_variant))):
        fn(inp, EventLedger())  # eager first call: plans, kernel attributes, tensor maps
        led = EventLedger(external=True)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            fn(inp, led)
        reps = []
        for r in range(runs + 2):
            graph.replay()
            if r >= 2:
                reps.append(led.snapshot())
        del graph
        st = aggregate(reps)
        op = st.operation_ns_mean
        pack = st.phase_ns_mean[Phase.IN_PACKING] + (st.phase_ns_mean[Phase.PRE_REORDER]
                                                    if name == "im2col_gemm" else 0.0)
        out[name] = {"operation_us": op / 1e3,
                     "gflops": algos.flop_count(d) / (op * 1e-9) / 1e9 if op else None,
                     "pack_share": pack / op if op else None,
                     "phases_us": {p.name.lower(): st.phase_ns_mean[p] / 1e3 for p in Phase
                                   if st.calls[p]},
                     "calls": {p.name.lower(): st.calls[p] for p in Phase if st.calls[p]},
                     "timing": "CUDA graph replay, external phase events"}
    torch.cuda.synchronize()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

"""BASELINE.json config 5: the synthetic convSet sweep on N GPUs.

    python tools/sweep.py --sample 400 --modes fused,baseline,main --out sweep_out
    python tools/sweep.py --gpus 8 --out sweep_out        # 8 ranks, one per GPU
    python tests/sweep_parity.py --out sweep_out          # the same sweep + CPU-oracle parity

Ops are independent, so ranks split them by LPT on the predicted roofline time (no
collective on the data path; gloo carries only the final gather).  `--gpus N` starts the
N ranks itself (paper_2407_10730_b200/launch.py); under torchrun it runs as the given rank.
Every rank generates each op's inputs once with make_inputs (bit-identical to the
reference harness), uploads them, and runs every mode on them through the package harness
(run_single: warmups, then measured runs on a CUDA-event ledger).  Duplicate ops (same
key, hence the same inputs) are adjacent and share one upload; each is still timed as its
own indexed op.  Rank 0 writes

  <out>/results_<mode>.csv   reference results schema (report.py:21-27), sweep order
  <out>/summary.json         per mode: GFLOP/s p10/p50/p90, roofline-fraction
                             distribution, pack share of the stepwise paths, status
                             counts, per-rank device-time makespan and the aggregate
                             GFLOP/s it implies (+ parity, when a checker ran)

--sample K keeps a seeded, FLOP-stratified subset of K ops.  --device-inputs draws the same
distribution on the GPU instead (not bit-identical to make_inputs; no parity check).

A `checker` (run(args, checker)) sees every op's outputs: tests/sweep_parity.py passes
the CPU-oracle one.  This tool never imports the oracle itself.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np

from paper_2407_10730_b200 import algos, configs, harness, report, roofline
from paper_2407_10730_b200.descriptor import flop_count, key_of
from paper_2407_10730_b200.launch import ensure_ranks
from paper_2407_10730_b200.shard import lpt_assign
from paper_2407_10730_b200.timing import Phase

LAUNCH_FLOOR_S = 5e-6  # per-op floor added to the roofline for LPT balance


def stratified_sample(descs, k: int, seed: int) -> list[int]:
    """k indices spread evenly over the FLOP-sorted sweep (seeded pick inside each stratum)."""
    if k >= len(descs):
        return list(range(len(descs)))
    order = sorted(range(len(descs)), key=lambda i: flop_count(descs[i]))
    rng = random.Random(seed)
    edges = np.linspace(0, len(order), k + 1).astype(int)
    return sorted(order[rng.randrange(a, b)] for a, b in zip(edges[:-1], edges[1:]) if b > a)


def predicted_s(desc, peaks) -> float:
    return roofline.conv_roofline(desc, algos.FUSED_DEFAULT_VARIANT, peaks)["t_roofline_s"] + LAUNCH_FLOOR_S


def pack_share(o, mode: str) -> float | None:
    if o.stats is None or not o.stats.operation_ns_mean:
        return None
    m = o.stats.phase_ns_mean
    pack = m[Phase.IN_PACKING] + (m[Phase.PRE_REORDER] if mode == "baseline" else 0.0)
    return pack / o.stats.operation_ns_mean


def pct(vals, q):
    return float(np.percentile(vals, q)) if vals else None


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=0,
                    help="ranks to start (one per GPU); 0: the torchrun environment, else 1")
    ap.add_argument("--opset", choices=["synthetic", "models"], default="synthetic",
                    help="synthetic: BASELINE config 5; models: configs/model_ops.json "
                         "(torchvision layers, tools/model_ops.py)")
    ap.add_argument("--ops", type=int, default=configs.SWEEP_SIZE)
    ap.add_argument("--seed", type=int, default=0, help="sweep generator seed")
    ap.add_argument("--data-seed", type=int, default=0, help="make_inputs seed")
    ap.add_argument("--sample", type=int, default=0, help="stratified subset size (0: all)")
    ap.add_argument("--modes", default="fused,baseline,main")
    ap.add_argument("--warmups", type=int, default=3)
    ap.add_argument("--runs", type=int, default=10)
    ap.add_argument("--variant", default=None, help=f"stepwise variant (default {algos.DEFAULT_VARIANT})")
    ap.add_argument("--fused-variant", default=algos.FUSED_AUTO)
    ap.add_argument("--device-inputs", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="time each op as a replayed CUDA graph (kernels without host launch gaps)")
    ap.add_argument("--max-gflop", type=float, default=0.0, help="skip larger ops (0: none)")
    ap.add_argument("--min-gflop", type=float, default=0.0, help="skip smaller ops")
    ap.add_argument("--out", default="sweep_out")
    ap.add_argument("--verbose", action="store_true", help="print every op key before it runs")
    ap.add_argument("--limit", type=int, default=0, help="diagnostics: run at most N ops per rank")
    ap.add_argument("--dry-run", action="store_true",
                    help="the multi-rank plumbing on CPU (gloo): LPT partition, per-rank rows with "
                         "the predicted time standing in for a measurement, gather, rank-0 outputs")
    return ap


def select_ops(args):
    """(descriptors, indices to run, model-op metadata or None)."""
    model_ops = None
    if args.opset == "models":
        from paper_2407_10730_b200.descriptor import parse_key
        model_ops = json.loads((Path(__file__).resolve().parent.parent / "configs" /
                                "model_ops.json").read_text())
        descs = [parse_key(k) for k in model_ops["unique"]]
    else:
        descs = configs.sweep(args.ops, args.seed)
    idx = stratified_sample(descs, args.sample, args.seed) if args.sample else list(range(len(descs)))
    if args.max_gflop > 0:
        idx = [i for i in idx if flop_count(descs[i]) <= args.max_gflop * 1e9]
    if args.min_gflop > 0:
        idx = [i for i in idx if flop_count(descs[i]) > args.min_gflop * 1e9]
    return descs, idx, model_ops


def run(args, checker=None, ranks=None) -> int:
    """The sweep on this rank; `checker` (optional) gets every op's outputs:
    checker.check(desc, host_inputs, [(index, mode, output), ...]) once per unique key,
    checker.finish() -> {(index, mode): result dict} on every rank after the last op."""
    rank, world, local = (ranks.rank, ranks.world, ranks.local) if ranks else (0, 1, 0)
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    if not args.dry_run:
        torch.cuda.set_device(local)
    if checker is not None and args.device_inputs:
        raise SystemExit("a parity check needs make_inputs host data (drop --device-inputs)")

    descs, idx, model_ops = select_ops(args)
    peaks = roofline.load_peaks()
    cost = [predicted_s(descs[i], peaks) for i in idx]
    mine = [idx[j] for j in lpt_assign(cost, world)[rank]]
    # duplicates adjacent (one upload per key); the largest ops first, so the slowest CPU
    # oracle jobs of a checker start early
    mine.sort(key=lambda i: (-flop_count(descs[i]), key_of(descs[i]), i))
    if args.limit:
        mine = mine[:args.limit]
    modes = [m for m in args.modes.split(",") if m]
    cfgs = {m: harness.RunConfig(mode=m, warmups=args.warmups, runs=args.runs,
                                 seed=args.data_seed, graph=args.graph,
                                 variant=args.fused_variant if m == "fused"
                                 else (args.variant or algos.DEFAULT_VARIANT)) for m in modes}

    local_rows: dict[str, list] = {m: [] for m in modes}
    busy = {m: 0.0 for m in modes}
    t0 = time.time()
    n = 0
    while args.dry_run and n < len(mine):  # no GPU: predicted times stand in for measurements
        from paper_2407_10730_b200.timing import _report, aggregate
        i = mine[n]
        d = descs[i]
        for m in modes:
            rf = roofline.conv_roofline(d, algos.resolve_variant(d, cfgs[m].variant), peaks)
            el = [0] * len(Phase)
            calls = [0] * len(Phase)
            el[Phase.IN_MICROKERNEL] = int(predicted_s(d, peaks) * 1e9)
            calls[Phase.IN_MICROKERNEL] = 1
            o = harness.RunOutcome(key=key_of(d), mode=m, runs=1, warmups=0, status="ok",
                                   stats=aggregate([_report(el, calls)]), detail="dry run")
            t_op = o.stats.operation_ns_mean * 1e-9
            busy[m] += t_op
            local_rows[m].append({"index": i, "record": report.outcome_record(o), "status": o.status,
                                  "flops": rf["flops"], "t_s": t_op, "t_min_s": t_op,
                                  "roofline_s": rf["t_roofline_s"], "pack_share": None, "detail": o.detail})
        n += 1
    while n < len(mine):
        d = descs[mine[n]]
        group = [mine[n]]
        while n + len(group) < len(mine) and descs[mine[n + len(group)]] == d:
            group.append(mine[n + len(group)])
        if args.device_inputs:
            host, dev = None, harness.device_inputs(d, cfgs[modes[0]])
        else:
            host = harness.make_inputs(d, cfgs[modes[0]])
            dev = harness.to_device(host)
        outs = []
        for i in group:
            for m in modes:
                if args.verbose:
                    print(f"[{m} {n}] {i} {descs[i]}", flush=True)
                o = harness.run_single(d, cfgs[m], inputs_fn=lambda *_: dev,
                                       keep_output=checker is not None)
                rf = roofline.conv_roofline(d, algos.resolve_variant(d, cfgs[m].variant), peaks)
                t_op = o.stats.operation_ns_mean * 1e-9 if o.stats else None
                if t_op:
                    busy[m] += t_op
                local_rows[m].append({
                    "index": i, "record": report.outcome_record(o), "status": o.status,
                    "flops": rf["flops"], "t_s": t_op,
                    "t_min_s": o.stats.operation_ns_min * 1e-9 if o.stats else None,
                    "roofline_s": rf["t_roofline_s"], "pack_share": pack_share(o, m),
                    "detail": o.detail})
                if o.output is not None:
                    outs.append((i, m, o.output))
        if checker is not None:
            checker.check(d, host, outs)
        del outs, dev
        n += len(group)
        if rank == 0 and (n // 50) != ((n - len(group)) // 50):
            extra = checker.progress() if checker is not None else ""
            print(f"[rank0] {n}/{len(mine)} ops, {time.time() - t0:.0f} s {extra}", flush=True)
    if not args.dry_run:
        torch.cuda.empty_cache()
    parity = checker.finish() if checker is not None else None

    gathered = [None] * world
    payload = {"rows": local_rows, "busy": busy, "n": len(mine), "parity": parity}
    if dist is not None:
        dist.all_gather_object(gathered, payload)
    else:
        gathered = [payload]
    if rank == 0:
        write_outputs(args, descs, idx, modes, gathered, model_ops, peaks, world,
                      time.time() - t0, checker)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def write_outputs(args, descs, idx, modes, gathered, model_ops, peaks, world, wall_s, checker):
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    summary = {"ops_total": len(descs), "ops_run": len(idx), "sweep_seed": args.seed,
               "data_seed": args.data_seed, "sample": args.sample, "world": world,
               "wall_s": wall_s,
               "inputs": "device (torch.rand, not make_inputs bits)" if args.device_inputs
               else "make_inputs (bit-identical to the reference), uploaded once per op key",
               "warmups": args.warmups, "runs": args.runs, "peaks": peaks,
               "timing": "dry run: predicted times, no GPU" if args.dry_run else
               "CUDA-graph replay per op (device phases, no host launch gaps)"
               if args.graph else "eager calls (device phases include launch latency)",
               "modes": {}}
    parity = {}
    for g in gathered:
        parity.update(g.get("parity") or {})
    for m in modes:
        rows = sorted((r for g in gathered for r in g["rows"][m]), key=lambda r: r["index"])
        report.write_results_csv([r["record"] for r in rows], out / f"results_{m}.csv")
        ok = [r for r in rows if r["status"] == "ok" and r["t_s"]]
        gfs = [r["flops"] / r["t_s"] / 1e9 for r in ok]
        frac = [r["roofline_s"] / r["t_s"] for r in ok]
        shares = [r["pack_share"] for r in ok if r["pack_share"] is not None]
        makespan = max(g["busy"][m] for g in gathered)
        flops = sum(r["flops"] for r in ok)
        summary["modes"][m] = {
            "variant": args.fused_variant if m == "fused" else (args.variant or algos.DEFAULT_VARIANT),
            "status": {s: sum(r["status"] == s for r in rows) for s in
                       ("ok", "skipped_unsupported", "failed")},
            "gflops_p10_p50_p90": [pct(gfs, 10), pct(gfs, 50), pct(gfs, 90)],
            "roofline_frac_p10_p50_p90": [pct(frac, 10), pct(frac, 50), pct(frac, 90)],
            "pack_share_p10_p50_p90": [pct(shares, 10), pct(shares, 50), pct(shares, 90)]
            if m != "fused" else None,
            "total_tflop": flops / 1e12,
            "device_makespan_s": makespan,
            "aggregate_tflops": flops / makespan / 1e12 if makespan else None,
            "per_rank_busy_s": [g["busy"][m] for g in gathered],
            "failed": [(r["index"], r["detail"]) for r in rows if r["status"] == "failed"][:20],
        }
        if checker is not None:
            summary["modes"][m]["parity"] = checker.summarize(
                m, [(r["index"], key_of(descs[r["index"]]), r["status"]) for r in rows], parity)
    if checker is not None:
        checker.write_table(out / "parity.csv", descs, parity)
        summary["parity_check"] = checker.describe()
    if model_ops is not None:  # per-model conv time: every layer, in network order
        t_of = {m: {key_of(descs[r["index"]]): r["t_s"] for g in gathered for r in g["rows"][m]}
                for m in modes}
        summary["opset"] = model_ops["source"]
        summary["models"] = {
            name: {"layers": len(mo["layers"]),
                   **{f"{m}_conv_ms": (sum(t_of[m].get(k) or 0.0 for k in mo["layers"]) * 1e3
                                       if all(t_of[m].get(k) for k in mo["layers"]) else None)
                      for m in modes}}
            for name, mo in model_ops["models"].items()}
    (out / "summary.json").write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps({m: {k: v for k, v in s.items() if k != "failed"}
                      for m, s in summary["modes"].items()}, indent=1))


def main(argv=None, checker_factory=None, script=None, relaunch_argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    args = parser().parse_args(argv)
    gpus = args.gpus or int(os.environ.get("WORLD_SIZE", 1))
    ranks = ensure_ranks(gpus, script or str(Path(__file__).resolve()),
                         argv if relaunch_argv is None else relaunch_argv)
    if isinstance(ranks, int):  # the relaunched ranks ran; propagate their exit code
        return ranks
    checker = checker_factory(args, ranks) if checker_factory else None
    return run(args, checker, ranks)


if __name__ == "__main__":
    sys.exit(main())

"""The N>1 path on CPU: 2 ranks over gloo (127.0.0.1), exercising the same sharding,
max-over-ranks timing and result gather the GPU runs use over NCCL.  The per-rank conv
here is the CPU oracle standing in for the GPU kernel, which lets the test check that
batch-sharded results reassemble into the unsharded convolution."""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle import conv_oracle as orc
    from paper_2407_10730_b200 import shard
    from paper_2407_10730_b200.configs import sweep
    from paper_2407_10730_b200.descriptor import ConvDescriptor, flop_count

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # batch sharding of one op: each rank convolves its slice with replicated weights
        d = ConvDescriptor(batch=5, in_channels=3, in_h=9, in_w=9, out_channels=4, k_h=3, k_w=3,
                           pad_h=1, pad_w=1, has_bias=True)
        x, w, b = orc.make_inputs(d, 0)
        start, count = shard.batch_shard(d.batch, world, rank)
        mine = shard.shard_descriptor(d, world, rank)
        y_part = orc.conv_direct_naive(mine, x[start:start + count], w, b)
        parts = shard.gather_to_rank0((start, y_part), dist)
        # sweep sharding: every rank derives the same LPT partition without talking
        s = sweep(200, seed=3)
        part = shard.sweep_partition(s, world, flop_count)[rank]
        all_parts = shard.gather_to_rank0(part, dist)
        t = shard.max_over_ranks(float(rank + 1), dist)
        tot = shard.sum_over_ranks(float(flop_count(mine)), dist)
        if rank == 0:
            parts.sort(key=lambda p: p[0])
            y = np.concatenate([p[1] for p in parts], axis=0)
            full = orc.conv_direct_naive(d, x, w, b)
            flat = sorted(i for p in all_parts for i in p)
            q.put(dict(equal=bool(np.array_equal(y, full)), cover=flat == list(range(200)),
                       disjoint=len(flat) == len(set(flat)), tmax=t,
                       flops=tot == flop_count(d)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0, "worker failed"
    res = q.get(timeout=10)
    assert res == dict(equal=True, cover=True, disjoint=True, tmax=2.0, flops=True), res


@pytest.mark.parametrize("n,world", [(128, 8), (16, 8), (5, 2), (3, 4)])
def test_batch_shard_partitions(n, world):
    from paper_2407_10730_b200.shard import batch_shard
    spans = [batch_shard(n, world, r) for r in range(world)]
    assert sum(c for _, c in spans) == n
    assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1

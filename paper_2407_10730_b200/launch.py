"""One process per GPU: the launcher bench.py and tools/sweep.py share.

`python bench.py --gpus N` (or tools/sweep.py --gpus N) with no torch.distributed
environment re-executes itself under `torch.distributed.run` with N local ranks on
127.0.0.1; under torchrun (RANK / WORLD_SIZE / LOCAL_RANK set by the driver) it runs as
the given rank.  A WORLD_SIZE that disagrees with --gpus is an error, never silently
ignored.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys
from dataclasses import dataclass


@dataclass(frozen=True)
class Ranks:
    rank: int
    world: int
    local: int


def env_ranks() -> Ranks | None:
    """The torchrun rank environment, or None outside one."""
    if "WORLD_SIZE" not in os.environ:
        return None
    rank = int(os.environ.get("RANK", 0))
    return Ranks(rank, int(os.environ["WORLD_SIZE"]), int(os.environ.get("LOCAL_RANK", rank)))


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_cmd(nproc: int, script: str, argv: list[str], port: int | None = None) -> list[str]:
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
            f"--master-port={port or free_port()}", script, *argv]


def ensure_ranks(gpus: int, script: str, argv: list[str]) -> Ranks | int:
    """Ranks of this process, or the exit code of a relaunch that already ran them.

    * inside torchrun: WORLD_SIZE must equal `gpus` (ValueError otherwise);
    * outside, gpus == 1: rank 0 of 1;
    * outside, gpus > 1: run `script argv` under torch.distributed.run with `gpus` local
      ranks and return its exit code (the caller exits with it)."""
    if gpus < 1:
        raise ValueError(f"--gpus must be >= 1, got {gpus}")
    r = env_ranks()
    if r is not None:
        if r.world != gpus:
            raise ValueError(f"--gpus {gpus} but WORLD_SIZE={r.world}: launch one rank per GPU "
                             f"(torchrun --nproc-per-node {gpus}) or drop the torchrun wrapper")
        return r
    if gpus == 1:
        return Ranks(0, 1, 0)
    return subprocess.call(relaunch_cmd(gpus, script, argv))

"""Multi-GPU plumbing: one process per GPU, work sharded by view or by frame.

Views of one MVD frame are independent and frames are
independent (pure functions, synthesis.py:9), so the path shards without any
per-pixel collective:

* ``shard`` — contiguous block of views (c2, c4) or round-robin frames (c3)
  for a rank;
* ``broadcast_frame`` — the one real exchange: the live MVD frame (RGB + u16
  depth + validity per camera, 6 B/px) arriving at one rank is replicated to
  all ranks with one NCCL broadcast per tensor over NVLink (gloo on CPU for
  the host tests);
* ``max_over_ranks`` — device-timed step times reduced with MAX, the only
  honest multi-GPU clock.

Works on any torch.distributed backend; nothing here touches the per-pixel
path.
"""

from __future__ import annotations

import os
from typing import List, Sequence

import torch
import torch.distributed as dist


def world() -> tuple:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str | None = None) -> tuple:
    rank, ws, local = world()
    if ws > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend, rank=rank, world_size=ws)
    return rank, ws, local


def shard(n_items: int, world_size: int, rank: int, mode: str = "block") -> List[int]:
    """Indices rank ``rank`` owns: ``block`` = contiguous near-equal blocks
    (views), ``cyclic`` = i mod world_size (frames)."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("bad rank/world size")
    if mode == "cyclic":
        return list(range(rank, n_items, world_size))
    if mode != "block":
        raise ValueError(f"unknown shard mode {mode!r}")
    base, extra = divmod(n_items, world_size)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def broadcast_frame(tensors: Sequence[torch.Tensor], src: int = 0) -> None:
    """Replicate the live frame's tensors from ``src`` to every rank, in place."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return
    for t in tensors:
        # as raw bytes: NCCL and gloo lack some raster dtypes (e.g. int16 mm)
        dist.broadcast(t.reshape(-1).view(torch.uint8), src=src)


def max_over_ranks(value: float) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()

"""Multi-GPU plumbing: one process per GPU, work sharded by view or by frame.

Views of one MVD frame are independent and frames are
independent (pure functions, synthesis.py:9), so the path shards without any
per-pixel collective:

* ``shard`` — contiguous block of views (c2, c4) or round-robin frames (c3)
  for a rank;
* ``pack_frame`` / ``broadcast_frame`` — the one real exchange: the live MVD
  frame (RGB + u16 depth + validity per camera, 6 B/px) arriving at one rank,
  packed into one flat buffer, is replicated to all ranks with a single NCCL
  broadcast over NVLink (gloo on CPU for the host tests);
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


def pack_frame(tensors: Sequence[torch.Tensor], device=None):
    """Copy a frame's tensors into ONE flat byte buffer (16-byte aligned
    slices) and return (flat, views): the views have the tensors' dtypes and
    shapes, so the frame is replicated with a single broadcast of `flat`."""
    sizes = [t.numel() * t.element_size() for t in tensors]
    offs, total = [], 0
    for n in sizes:
        offs.append(total)
        total += (n + 15) // 16 * 16
    dev = tensors[0].device if device is None else device
    flat = torch.empty(total, dtype=torch.uint8, device=dev)
    views = []
    for t, o, n in zip(tensors, offs, sizes):
        v = flat[o:o + n].view(t.dtype).view(t.shape)
        v.copy_(t)
        views.append(v)
    return flat, views


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


def gather_over_ranks(value: float) -> List[float]:
    """``value`` of every rank, in rank order (a list of one without a group)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(value)]
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()

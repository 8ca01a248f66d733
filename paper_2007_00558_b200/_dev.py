"""Device-buffer plumbing (torch is used only for memory and streams)."""

from __future__ import annotations

import numpy as np
import torch

# uint16 rasters travel as int16 (same bytes; torch's uint16 support is partial)
_DT = {np.uint8: torch.uint8, np.uint16: torch.int16, np.int32: torch.int32,
       np.int64: torch.int64, np.float32: torch.float32, np.float64: torch.float64}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2007_00558_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def upload(a, dtype) -> torch.Tensor:
    """Host array / device tensor -> contiguous device tensor of ``dtype``."""
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.uint16:
            a = a.view(torch.int16)
        t = a.to(device=device(), dtype=_DT[np.dtype(dtype).type])
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    if any(st < 0 for st in arr.strides):  # e.g. a reversed 1-element view
        arr = arr.copy()
    if arr.dtype == np.uint16:
        arr = arr.view(np.int16)
    return torch.from_numpy(arr).to(device())


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(tuple(shape), dtype=_DT[np.dtype(dtype).type], device=device())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(tuple(shape), dtype=_DT[np.dtype(dtype).type], device=device())


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def host(t: torch.Tensor, dtype=None) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view(dtype) if dtype is not None else a


def check_out(t, dtype, what: str, shape=None, dev: int | None = None) -> None:
    """An output tensor the library writes: CUDA, ``dtype``, contiguous, and
    (when given) exactly ``shape``; else ValueError before any kernel runs."""
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise ValueError(f"{what} must be a CUDA tensor")
    want = device() if dev is None else torch.device("cuda", dev)
    if t.device != want:
        raise ValueError(f"{what} is on {t.device}, the renderer on {want}")
    if t.dtype != dtype:
        raise ValueError(f"{what} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what} has shape {tuple(t.shape)}, expected {tuple(shape)}")

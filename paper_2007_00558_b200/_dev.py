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

"""Edge-server depth preprocessing on B200 — drop-ins for the reference calls.

* ``bilateral_close_holes``  -> ``fvv.depthproc.bilateral_close_holes``
  (depthproc.py:171-224), kernel K1 via ``fvv_bilateral_close_holes``;
* ``depth_from_millimeters`` -> ``fvv.core.depth_from_millimeters``
  (core.py:260-269), kernel K0 via ``fvv_decode_mm``.

The capture-server functions of ``fvv.depthproc`` (correction, BG model, BG
removal) are not on the edge-server path and are not provided.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _native
from .types import ColorFrame, DepthFrame, Validity


def bilateral_close_holes(depth, guide, radius: int = 2, sigma_spatial: float = 2.0,
                          sigma_range: float = 10.0, min_valid_neighbors: int = 6):
    """Joint-bilateral fill of Invalid pixels from >= ``min_valid_neighbors`` Valid ones.

    Returns ``depth`` itself when it holds no Invalid pixel, like the
    reference (depthproc.py:188-190).
    """
    if (guide.height, guide.width) != (depth.height, depth.width):
        raise ValueError("guide dimensions do not match the depth frame")
    val = depth.validity
    if isinstance(val, np.ndarray) and not (val == Validity.INVALID).any():
        return depth
    ctx = _native.context()
    W, H = int(depth.width), int(depth.height)
    d = _dev.upload(depth.depth, np.float32)
    v = _dev.upload(val, np.uint8)
    g = _dev.upload(guide.pixels, np.uint8)
    out_d = _dev.empty((H, W), np.float32)
    out_v = _dev.empty((H, W), np.uint8)
    holes = _dev.zeros((1,), np.int32)
    ctx.call("fvv_bilateral_close_holes", d.data_ptr(), v.data_ptr(), g.data_ptr(), W, H,
             int(radius), float(sigma_spatial), float(sigma_range), int(min_valid_neighbors),
             out_d.data_ptr(), out_v.data_ptr(), holes.data_ptr())
    if int(holes.item()) == 0:
        return depth
    return DepthFrame(W, H, _dev.host(out_d), _dev.host(out_v), depth.timestamp_us)


def depth_from_millimeters(mm, validity, timestamp_us: int = 0) -> DepthFrame:
    """u16 mm raster + validity -> DepthFrame (fp32 true division by 1000)."""
    mm = np.asarray(mm) if not isinstance(mm, torch.Tensor) else mm
    H, W = mm.shape
    ctx = _native.context()
    m = _dev.upload(mm, np.uint16)
    v = _dev.upload(validity, np.uint8)
    out_d = _dev.empty((H, W), np.float32)
    out_v = _dev.empty((H, W), np.uint8)
    ctx.call("fvv_decode_mm", m.data_ptr(), v.data_ptr(), W, H, out_d.data_ptr(),
             out_v.data_ptr())
    return DepthFrame(W, H, _dev.host(out_d), _dev.host(out_v), timestamp_us)


__all__ = ["bilateral_close_holes", "depth_from_millimeters", "ColorFrame", "DepthFrame"]

"""Edge-server depth preprocessing on B200 — drop-ins for the reference calls.

* ``bilateral_close_holes``  -> ``fvv.depthproc.bilateral_close_holes``
  (depthproc.py:171-224), kernel K1 via ``fvv_bilateral_close_holes``;
* ``depth_from_millimeters`` -> ``fvv.core.depth_from_millimeters``
  (core.py:260-269), kernel K0 via ``fvv_decode_mm``.

Capture-server side (widened after the edge-server
path): ``CorrectionModel`` / ``correct_depth`` (depthproc.py:30-84),
``GaussianBgModel`` / ``bg_train`` / ``classify_fg`` (depthproc.py:91-149) and
``remove_bg_depth`` (depthproc.py:152-164), on the GPU. The control-point
fit (``fit_depth_correction``) is a host least-squares over a few hundred
points and stays in the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

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
    if int(radius) > 0:
        ctx.range_weights(sigma_range)
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




# ---------------------------------------------------------------------------
# capture-server chain: depthproc.py:30-164 drop-ins


class DegenerateFitError(ValueError):
    """A correction fit without enough distinct control depths (depthproc.py:22)."""


class UntrainedModelError(RuntimeError):
    """Classification on a BG model still in warm-up (depthproc.py:26)."""


@dataclass(frozen=True)
class CorrectionModel:
    """Quadratic depth correction z_post = (alpha * z + beta) * z (depthproc.py:30-41)."""

    alpha: float
    beta: float
    residual_rms: float = 0.0

    def __post_init__(self):
        if not all(math.isfinite(x) for x in (self.alpha, self.beta, self.residual_rms)):
            raise ValueError("correction model parameters must be finite")


def correct_depth(frame, model) -> DepthFrame:
    """Quadratic correction of every Valid pixel on the GPU (depthproc.py:67-84)."""
    ctx = _native.context()
    W, H = int(frame.width), int(frame.height)
    d = _dev.upload(frame.depth, np.float32)
    v = _dev.upload(frame.validity, np.uint8)
    od = _dev.empty((H, W), np.float32)
    ov = _dev.empty((H, W), np.uint8)
    ctx.call("fvv_correct_depth", d.data_ptr(), v.data_ptr(), W, H, float(model.alpha),
             float(model.beta), od.data_ptr(), ov.data_ptr())
    return DepthFrame(W, H, _dev.host(od), _dev.host(ov), frame.timestamp_us)


@dataclass
class GaussianBgModel:
    """Per-pixel running Gaussian of the BG colour (depthproc.py:91-118).

    ``mean`` / ``var`` are host float64 (H, W, 3) arrays like the reference's;
    ``bg_train`` / ``classify_fg`` run on the GPU.
    """

    width: int
    height: int
    warmup_frames: int = 30
    learning_rate: float = 0.02
    threshold: float = 3.5
    var_floor: float = 4.0
    frames_trained: int = 0
    mean: np.ndarray = field(default=None, repr=False)
    var: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        if self.mean is None:
            self.mean = np.zeros((self.height, self.width, 3), dtype=np.float64)
        if self.var is None:
            self.var = np.full((self.height, self.width, 3), self.var_floor, dtype=np.float64)

    @property
    def trained(self) -> bool:
        return self.frames_trained >= self.warmup_frames


def bg_train(model: GaussianBgModel, frame) -> GaussianBgModel:
    """Warm-up update of the running mean / variance (depthproc.py:121-136)."""
    if (frame.height, frame.width) != (model.height, model.width):
        raise ValueError("frame dimensions do not match the model")
    ctx = _native.context()
    rgb = _dev.upload(frame.pixels, np.uint8)
    mean = _dev.upload(model.mean, np.float64)
    var = _dev.upload(model.var, np.float64)
    ctx.call("fvv_bg_train", rgb.data_ptr(), model.width, model.height, mean.data_ptr(),
             var.data_ptr(), int(model.frames_trained == 0), float(model.learning_rate),
             float(model.var_floor))
    model.mean[:] = _dev.host(mean)
    model.var[:] = _dev.host(var)
    model.frames_trained += 1
    return model


def classify_fg(model: GaussianBgModel, frame) -> np.ndarray:
    """FG mask: sum_c (x - mu)^2 / sigma^2 > tau^2 (depthproc.py:139-149)."""
    if not model.trained:
        raise UntrainedModelError(
            f"model warm-up incomplete ({model.frames_trained}/{model.warmup_frames})")
    if (frame.height, frame.width) != (model.height, model.width):
        raise ValueError("frame dimensions do not match the model")
    ctx = _native.context()
    rgb = _dev.upload(frame.pixels, np.uint8)
    mean = _dev.upload(model.mean, np.float64)
    var = _dev.upload(model.var, np.float64)
    mask = _dev.empty((model.height, model.width), np.uint8)
    ctx.call("fvv_classify_fg", rgb.data_ptr(), mean.data_ptr(), var.data_ptr(), model.width,
             model.height, float(model.threshold), mask.data_ptr())
    return _dev.host(mask).astype(bool)


def remove_bg_depth(depth, mask) -> DepthFrame:
    """BG-mask pixels become Background with depth 0 (depthproc.py:152-164)."""
    mask = np.asarray(mask)
    if mask.shape != (depth.height, depth.width):
        raise ValueError("mask dimensions do not match the depth frame")
    ctx = _native.context()
    W, H = int(depth.width), int(depth.height)
    d = _dev.upload(depth.depth, np.float32)
    v = _dev.upload(depth.validity, np.uint8)
    m = _dev.upload(mask.astype(bool), np.uint8)
    od = _dev.empty((H, W), np.float32)
    ov = _dev.empty((H, W), np.uint8)
    ctx.call("fvv_remove_bg_depth", d.data_ptr(), v.data_ptr(), m.data_ptr(), W, H,
             od.data_ptr(), ov.data_ptr())
    return DepthFrame(W, H, _dev.host(od), _dev.host(ov), depth.timestamp_us)


__all__ = ["bilateral_close_holes", "depth_from_millimeters", "CorrectionModel", "correct_depth",
           "GaussianBgModel", "bg_train", "classify_fg", "remove_bg_depth",
           "UntrainedModelError", "DegenerateFitError", "ColorFrame", "DepthFrame"]

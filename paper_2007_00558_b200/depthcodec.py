"""12-bit depth decode on B200 — drop-ins for the edge-server half of ``fvv.depthcodec``.

* ``unpack_yuv420`` -> depthcodec.unpack_yuv420 (depthcodec.py:154-177, 213-222)
* ``dequantize12``  -> depthcodec.dequantize12 (depthcodec.py:113-138)
* ``decode_yuv420_depth`` -> both fused in one pass (kernel K0, the form the
  edge server runs, pipeline.py:469-472).

The encoder half (``quantize12`` / ``pack_yuv420`` and the fused
``capture_encode`` of the capture server's per-frame chain) is provided as
SURVEY.md §8f's rank-1 widening. The MED+Rice entropy coder (a sequential
bitstream) is not.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _native
from .types import DepthFrame, DepthRange

DISPARITY_MAX = 4095
CODE_BACKGROUND = 0
CODE_INVALID = 1
CODE_MIN_VALID = 2
LEVELS = 2 ** 12 - 3


@dataclass(frozen=True)
class DisparityMap12:
    """12-bit disparity raster with reserved codes 0/1 (depthcodec.py:32-45)."""

    width: int
    height: int
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.uint16)
        if v.shape != (self.height, self.width):
            raise ValueError(f"values shape {v.shape} != {self.height}x{self.width}")
        if v.size and v.max() > DISPARITY_MAX:
            raise ValueError("disparity values exceed 12 bits")
        object.__setattr__(self, "values", v)


@dataclass(frozen=True)
class Yuv420Image:
    """8-bit YUV420 planes (depthcodec.py:48-76)."""

    y: np.ndarray
    u: np.ndarray
    v: np.ndarray

    def __post_init__(self):
        y, u, v = (np.asarray(a, dtype=np.uint8) for a in (self.y, self.u, self.v))
        h, w = y.shape
        if h % 2 or w % 2:
            raise ValueError("YUV420 dimensions must be even")
        if u.shape != (h // 2, w // 2) or v.shape != (h // 2, w // 2):
            raise ValueError("chroma plane sizes inconsistent with luma")
        object.__setattr__(self, "y", y)
        object.__setattr__(self, "u", u)
        object.__setattr__(self, "v", v)

    @property
    def width(self) -> int:
        return self.y.shape[1]

    @property
    def height(self) -> int:
        return self.y.shape[0]


def _decode(img, range_: DepthRange):
    ctx = _native.context()
    H, W = img.y.shape
    y, u, v = (_dev.upload(a, np.uint8) for a in (img.y, img.u, img.v))
    d = _dev.empty((H, W), np.float32)
    val = _dev.empty((H, W), np.uint8)
    codes = _dev.empty((H, W), np.uint16)
    ctx.call("fvv_decode_yuv420_12", y.data_ptr(), u.data_ptr(), v.data_ptr(), W, H,
             float(range_.z_near), float(range_.z_far), d.data_ptr(), val.data_ptr(),
             codes.data_ptr())
    return d, val, codes


def unpack_yuv420(img: Yuv420Image) -> DisparityMap12:
    """Bit-exact inverse of the LSB fold + nibble interleave."""
    H, W = img.y.shape
    _, _, codes = _decode(img, DepthRange(1.0, 2.0))
    return DisparityMap12(W, H, _dev.host(codes, np.uint16))


def dequantize12(d: DisparityMap12, range_: DepthRange, timestamp_us: int = 0) -> DepthFrame:
    """Codes -> metric depth: code 0 Background, 1 Invalid, else the f64 inverse map."""
    ctx = _native.context()
    H, W = d.values.shape
    c = _dev.upload(d.values, np.uint16)
    z = _dev.empty((H, W), np.float32)
    val = _dev.empty((H, W), np.uint8)
    ctx.call("fvv_dequantize12", c.data_ptr(), W, H, float(range_.z_near),
             float(range_.z_far), z.data_ptr(), val.data_ptr())
    return DepthFrame(W, H, _dev.host(z), _dev.host(val), timestamp_us)


def decode_yuv420_depth(img: Yuv420Image, range_: DepthRange, timestamp_us: int = 0) -> DepthFrame:
    """``dequantize12(unpack_yuv420(img))`` in one kernel pass."""
    H, W = img.y.shape
    d, val, _ = _decode(img, range_)
    return DepthFrame(W, H, _dev.host(d), _dev.host(val), timestamp_us)


# ---------------------------------------------------------------------------
# encoder half: depthcodec.py:83-110, 180-193


def quantize12(depth, range_: DepthRange) -> DisparityMap12:
    """Metric depth -> 12-bit codes: 0 Background, 1 Invalid/out of band (depthcodec.py:83-110)."""
    ctx = _native.context()
    W, H = int(depth.width), int(depth.height)
    d = _dev.upload(depth.depth, np.float32)
    v = _dev.upload(depth.validity, np.uint8)
    codes = _dev.empty((H, W), np.uint16)
    ctx.call("fvv_quantize12", d.data_ptr(), v.data_ptr(), W, H, float(range_.z_near),
             float(range_.z_far), codes.data_ptr())
    return DisparityMap12(W, H, _dev.host(codes, np.uint16))


def pack_yuv420(d: DisparityMap12) -> Yuv420Image:
    """LSB fold + MSB nibble interleave into YUV420 (depthcodec.py:180-193)."""
    if d.width % 2 or d.height % 2:
        raise ValueError("disparity map dimensions must be even")
    ctx = _native.context()
    c = _dev.upload(d.values, np.uint16)
    y = _dev.empty((d.height, d.width), np.uint8)
    u = _dev.empty((d.height // 2, d.width // 2), np.uint8)
    v = _dev.empty((d.height // 2, d.width // 2), np.uint8)
    ctx.call("fvv_pack_yuv420", c.data_ptr(), d.width, d.height, y.data_ptr(), u.data_ptr(),
             v.data_ptr())
    return Yuv420Image(_dev.host(y), _dev.host(u), _dev.host(v))


def capture_encode(depth, color, range_: DepthRange, correction=None, bg_model=None):
    """CaptureServer.capture's chain (pipeline.py:384-397) in one kernel:
    correct_depth -> classify_fg -> remove_bg_depth -> quantize12 -> pack_yuv420.

    Returns (Yuv420Image, DisparityMap12)."""
    ctx = _native.context()
    W, H = int(depth.width), int(depth.height)
    if W % 2 or H % 2:
        raise ValueError("YUV420 dimensions must be even")
    d = _dev.upload(depth.depth, np.float32)
    v = _dev.upload(depth.validity, np.uint8)
    rgb = _dev.upload(color.pixels, np.uint8) if color is not None else None
    if bg_model is not None and not bg_model.trained:
        from .depthproc import UntrainedModelError
        raise UntrainedModelError("BG model warm-up incomplete")
    mean = _dev.upload(bg_model.mean, np.float64) if bg_model is not None else None
    var = _dev.upload(bg_model.var, np.float64) if bg_model is not None else None
    y = _dev.empty((H, W), np.uint8)
    u = _dev.empty((H // 2, W // 2), np.uint8)
    vv = _dev.empty((H // 2, W // 2), np.uint8)
    codes = _dev.empty((H, W), np.uint16)
    ctx.call("fvv_capture_encode", d.data_ptr(), v.data_ptr(), _dev.ptr(rgb), W, H,
             int(correction is not None),
             float(correction.alpha) if correction is not None else 0.0,
             float(correction.beta) if correction is not None else 0.0,
             _dev.ptr(mean), _dev.ptr(var),
             float(bg_model.threshold) if bg_model is not None else 0.0,
             float(range_.z_near), float(range_.z_far), y.data_ptr(), u.data_ptr(),
             vv.data_ptr(), codes.data_ptr())
    return (Yuv420Image(_dev.host(y), _dev.host(u), _dev.host(vv)),
            DisparityMap12(W, H, _dev.host(codes, np.uint16)))

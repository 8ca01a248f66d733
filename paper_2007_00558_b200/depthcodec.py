"""12-bit depth decode on B200 — drop-ins for the edge-server half of ``fvv.depthcodec``.

* ``unpack_yuv420`` -> depthcodec.unpack_yuv420 (depthcodec.py:154-177, 213-222)
* ``dequantize12``  -> depthcodec.dequantize12 (depthcodec.py:113-138)
* ``decode_yuv420_depth`` -> both fused in one pass (kernel K0, the form the
  edge server runs, pipeline.py:469-472).

The encoder half (``quantize12`` / ``pack_yuv420`` and the fused
``capture_encode`` of the capture server's per-frame chain) is provided as
SURVEY.md §8f's rank-1 widening; the MED + Golomb-Rice lossless plane codec
(``encode_lossless`` / ``decode_lossless``, the wire format of the depth
stream) as its rank-4 widening.
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


# ---------------------------------------------------------------------------
# Encoded frames and the MED + Golomb-Rice lossless codec (SURVEY.md §8f
# rank 4): depthcodec.py:225-267 (frame container, registry, errors) and
# 281-464 (plane codec). The MED prediction, zig-zag, Rice parameter choice
# and the bit stream run on the GPU (fvv_rice_encode_plane /
# fvv_rice_decode_plane); the per-plane header and the optional zlib stage
# around the stream are the reference's own struct / zlib calls on the host.

import struct  # noqa: E402
import zlib  # noqa: E402
import ctypes as C  # noqa: E402
from typing import Callable, Dict, Tuple  # noqa: E402

MEDIA_COLOR = 0
MEDIA_DEPTH = 1

CODEC_RAW = 0
CODEC_ZLIB = 1
CODEC_PRED_RICE = 2

_HEADER = struct.Struct(">BBHHQI")        # codec, media, width, height, timestamp, length
_PLANE_HEADER = struct.Struct(">BBIII")   # k, deflate flag, symbols, bytes, adler32


@dataclass(frozen=True)
class EncodedFrame:
    """depthcodec.EncodedFrame (depthcodec.py:236-259)."""

    media_type: int
    codec_id: int
    width: int
    height: int
    timestamp_us: int
    payload: bytes

    def serialize(self) -> bytes:
        return _HEADER.pack(self.codec_id, self.media_type, self.width, self.height,
                            self.timestamp_us, len(self.payload)) + self.payload

    @staticmethod
    def deserialize(data: bytes) -> "EncodedFrame":
        if len(data) < _HEADER.size:
            raise ValueError("encoded frame truncated")
        codec, media, w, h, ts, n = _HEADER.unpack_from(data)
        if len(data) != _HEADER.size + n:
            raise ValueError("encoded frame length mismatch")
        return EncodedFrame(media, codec, w, h, ts, data[_HEADER.size:])


class UnsupportedCodecError(ValueError):
    pass


class DecodeError(ValueError):
    pass


def _compress_plane(plane: np.ndarray) -> bytes:
    """depthcodec._compress_plane (depthcodec.py:373-383) with the MED + Rice
    stage on the GPU."""
    plane = np.ascontiguousarray(plane, dtype=np.uint8)
    H, W = plane.shape
    ctx = _native.context()
    x = _dev.upload(plane, np.uint8)
    bound = int(ctx.lib.fvv_rice_stream_bound(W, H))
    stream = _dev.empty((bound,), np.uint8)
    k, nbits = C.c_int32(), C.c_int64()
    ctx.call("fvv_rice_encode_plane", x.data_ptr(), W, H, stream.data_ptr(), C.byref(k),
             C.byref(nbits))
    raw = _dev.host(stream[:(nbits.value + 7) // 8]).tobytes()
    deflated = zlib.compress(raw, 6)
    blob, flag = (deflated, 1) if len(deflated) < len(raw) else (raw, 0)
    return _PLANE_HEADER.pack(k.value, flag, W * H, len(blob), zlib.adler32(plane.tobytes())) + blob


def _parse_plane(data: bytes, offset: int, shape):
    """Host half of depthcodec._decompress_plane (depthcodec.py:386-397): the
    plane header, the blob and the zlib stage. Returns (k, stream, adler32,
    new offset)."""
    if len(data) - offset < _PLANE_HEADER.size:
        raise DecodeError("plane header truncated")
    k, flag, n, blob_len, check = _PLANE_HEADER.unpack_from(data, offset)
    offset += _PLANE_HEADER.size
    blob = data[offset:offset + blob_len]
    if len(blob) != blob_len:
        raise DecodeError("plane blob truncated")
    offset += blob_len
    try:
        stream = zlib.decompress(blob) if flag else blob
    except zlib.error as e:
        raise DecodeError(f"payload does not decode: {e}") from None
    if n != shape[0] * shape[1]:
        raise DecodeError("plane symbol count mismatch")
    return k, stream, check, offset


def _decode_planes_dev(planes):
    """Rice + MED stage of several planes in ONE batched GPU call
    (fvv_rice_decode_planes; their recurrences run concurrently). `planes` is
    a list of (k, stream bytes, adler32, (H, W)); returns device tensors."""
    ctx = _native.context()
    n = len(planes)
    keep, outs = [], []
    for k, stream, _, (H, W) in planes:
        keep.append(_dev.upload(np.frombuffer(stream, dtype=np.uint8), np.uint8)
                    if stream else None)
        outs.append(_dev.empty((H, W), np.uint8))
    VP = C.c_void_p * n
    I64, I32 = C.c_int64 * n, C.c_int32 * n
    adlers, status = (C.c_uint32 * n)(), I32()
    ctx.call("fvv_rice_decode_planes", n, VP(*[_dev.ptr(t) for t in keep]),
             I64(*[len(p[1]) for p in planes]), I32(*[int(p[0]) for p in planes]),
             I32(*[int(p[3][1]) for p in planes]), I32(*[int(p[3][0]) for p in planes]),
             VP(*[t.data_ptr() for t in outs]), adlers, status)
    for i, (_, _, check, _) in enumerate(planes):
        if status[i]:
            raise DecodeError("rice stream truncated")
        if adlers[i] != check:
            raise DecodeError("plane checksum mismatch")
    return outs


def _decompress_plane_dev(data: bytes, offset: int, shape):
    """depthcodec._decompress_plane (depthcodec.py:386-409), GPU Rice + MED;
    returns (device plane tensor, new offset)."""
    k, stream, check, offset = _parse_plane(data, offset, shape)
    try:
        out = _decode_planes_dev([(k, stream, check, shape)])[0]
    except ValueError as e:
        raise DecodeError(str(e)) from None
    return out, offset


def _decompress_plane(data: bytes, offset: int, shape) -> Tuple[np.ndarray, int]:
    out, offset = _decompress_plane_dev(data, offset, shape)
    return _dev.host(out), offset


_COMPRESSORS: Dict[int, Tuple[Callable[[bytes], bytes], Callable[[bytes], bytes]]] = {
    CODEC_RAW: (lambda b: b, lambda b: b),
    CODEC_ZLIB: (lambda b: zlib.compress(b, 6), zlib.decompress),
}


def register_codec(codec_id: int, compress: Callable[[bytes], bytes],
                   decompress: Callable[[bytes], bytes]) -> None:
    """Register an alternative lossless byte compressor (depthcodec.py:416-421)."""
    if codec_id in _COMPRESSORS or codec_id == CODEC_PRED_RICE:
        raise ValueError(f"codec id {codec_id} already registered")
    _COMPRESSORS[codec_id] = (compress, decompress)


def _codec(codec_id: int):
    try:
        return _COMPRESSORS[codec_id]
    except KeyError:
        raise UnsupportedCodecError(f"codec id {codec_id} is not a byte-stream codec") from None


def encode_lossless(img: Yuv420Image, timestamp_us: int = 0,
                    codec_id: int = CODEC_PRED_RICE) -> EncodedFrame:
    """depthcodec.encode_lossless (depthcodec.py:435-443)."""
    if codec_id == CODEC_PRED_RICE:
        payload = b"".join(_compress_plane(p) for p in (img.y, img.u, img.v))
    else:
        compress, _ = _codec(codec_id)
        payload = compress(img.y.tobytes() + img.u.tobytes() + img.v.tobytes())
    return EncodedFrame(MEDIA_DEPTH, codec_id, img.width, img.height, timestamp_us, payload)


def decode_lossless_many(frames):
    """The YUV420 planes of several CODEC_PRED_RICE depth frames (e.g. every
    reference camera of a render tick) as device tensors, decoded in one
    batched GPU call: returns [(y, u, v), ...] (the form the edge server feeds
    K0, pipeline.py:469-472)."""
    planes, layout = [], []
    for frame in frames:
        if frame.codec_id != CODEC_PRED_RICE:
            raise UnsupportedCodecError("decode_lossless_many takes CODEC_PRED_RICE frames")
        w, h = frame.width, frame.height
        try:
            off = 0
            for shape in ((h, w), (h // 2, w // 2), (h // 2, w // 2)):
                k, stream, check, off = _parse_plane(frame.payload, off, shape)
                planes.append((k, stream, check, shape))
        except DecodeError:
            raise
        except Exception as e:
            raise DecodeError(f"payload does not decode: {e}") from e
        if off != len(frame.payload):
            raise DecodeError("trailing bytes after planes")
        layout.append(len(planes) - 3)
    try:
        outs = _decode_planes_dev(planes)
    except DecodeError:
        raise
    except ValueError as e:
        raise DecodeError(str(e)) from None
    return [tuple(outs[i:i + 3]) for i in layout]


def decode_lossless_planes(frame: EncodedFrame):
    """The three YUV420 planes of one CODEC_PRED_RICE depth frame as device
    tensors (one batched GPU call)."""
    return decode_lossless_many([frame])[0]


def decode_lossless(frame: EncodedFrame) -> Yuv420Image:
    """depthcodec.decode_lossless (depthcodec.py:446-470)."""
    w, h = frame.width, frame.height
    if frame.codec_id == CODEC_PRED_RICE:
        y, u, v = decode_lossless_planes(frame)
        return Yuv420Image(_dev.host(y), _dev.host(u), _dev.host(v))
    _, decompress = _codec(frame.codec_id)
    try:
        raw = decompress(frame.payload)
    except Exception as e:
        raise DecodeError(f"payload does not decode: {e}") from e
    if len(raw) != w * h + 2 * (w // 2) * (h // 2):
        raise DecodeError("decoded plane size mismatch")
    y = np.frombuffer(raw, dtype=np.uint8, count=w * h).reshape(h, w)
    cn = (w // 2) * (h // 2)
    u = np.frombuffer(raw, dtype=np.uint8, count=cn, offset=w * h).reshape(h // 2, w // 2)
    v = np.frombuffer(raw, dtype=np.uint8, count=cn, offset=w * h + cn).reshape(h // 2, w // 2)
    return Yuv420Image(y.copy(), u.copy(), v.copy())

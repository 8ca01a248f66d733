"""ctypes binding of the C oracle — TEST / BASELINE INFRASTRUCTURE ONLY.

``es_view`` has the same signature and result as ``fvv_oracle.es_view``
(mm decode -> bilateral hole fill -> synthesize_view, pipeline.py:514-547)
and is bit-identical to it on integer outputs (tests/test_oracle.py).
The foreign calls release the GIL, so a thread pool runs views in parallel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .build import LIB, build_oracle
from .fvv_oracle import Cam, blend_weight


class _Cam(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("R", C.c_double * 9), ("C", C.c_double * 3)]


class _Ref(C.Structure):
    _fields_ = [("cam", _Cam), ("rgb", C.c_void_p), ("live_depth", C.c_void_p),
                ("live_validity", C.c_void_p), ("bg_depth", C.c_void_p),
                ("bg_validity", C.c_void_p), ("weight", C.c_double)]


class _Cfg(C.Structure):
    _fields_ = [("splat_radius", C.c_int32), ("crack_fill_window", C.c_int32),
                ("depth_band_rel", C.c_double), ("hole_color", C.c_uint8 * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = C.CDLL(str(LIB))
        _lib.fo_decode_mm.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                      C.c_void_p]
        _lib.fo_bilateral.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                      C.c_int, C.c_double, C.c_double, C.c_int, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
        _lib.fo_bilateral.restype = C.c_long
        _lib.fo_synthesize_view.argtypes = [C.POINTER(_Cam), C.POINTER(_Ref), C.c_int,
                                            C.POINTER(_Cfg), C.c_void_p, C.c_void_p]
    return _lib


def _cam(c) -> _Cam:
    c = c if isinstance(c, Cam) else Cam(c)
    out = _Cam(c.width, c.height, c.fx, c.fy, c.cx, c.cy)
    out.R[:] = [float(x) for x in c.R.ravel()]
    out.C[:] = [float(x) for x in c.C]
    return out


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def decode_mm(mm, validity):
    mm = np.ascontiguousarray(mm, np.uint16)
    H, W = mm.shape
    d = np.empty((H, W), np.float32)
    v = np.empty((H, W), np.uint8)
    val = None if validity is None else np.ascontiguousarray(validity, np.uint8)
    lib().fo_decode_mm(_p(mm), None if val is None else _p(val), W, H, _p(d), _p(v))
    return d, v


_range_tables: dict = {}


def _range_table(sigma_range):
    """np.exp(-color_d2 * inv_2sr) over every integer color_d2 (depthproc.py:
    200,212), so the C restatement uses numpy's exp like the reference."""
    t = _range_tables.get(sigma_range)
    if t is None:
        inv_2sr = 1.0 / (2.0 * sigma_range ** 2)
        t = _range_tables[sigma_range] = np.exp(-np.arange(3 * 255 * 255 + 1, dtype=np.float64)
                                                * inv_2sr)
    return t


def bilateral_close_holes(depth, validity, rgb, radius=2, sigma_spatial=2.0, sigma_range=10.0,
                          min_valid_neighbors=6):
    depth = np.ascontiguousarray(depth, np.float32)
    validity = np.ascontiguousarray(validity, np.uint8)
    rgb = np.ascontiguousarray(rgb, np.uint8)
    H, W = depth.shape
    od = np.empty_like(depth)
    ov = np.empty_like(validity)
    lib().fo_bilateral(_p(depth), _p(validity), _p(rgb), W, H, radius, sigma_spatial,
                       sigma_range, min_valid_neighbors, _p(od), _p(ov),
                       _p(_range_table(sigma_range)))
    return od, ov


def synthesize_view(virtual, refs, cfg=None):
    cfg = dict(dict(splat_radius=1, crack_fill_window=3, mixing_epsilon=0.01,
                    depth_band_rel=0.02, hole_color=(0, 0, 0)), **(cfg or {}))
    if not refs:
        raise ValueError("need at least one reference camera")
    dst = Cam(virtual)
    arr = (_Ref * len(refs))()
    keep = []
    for j, s in enumerate(refs):
        bufs = [np.ascontiguousarray(s[k], dt) for k, dt in (
            ("rgb", np.uint8), ("live_depth", np.float32), ("live_validity", np.uint8),
            ("bg_depth", np.float32), ("bg_validity", np.uint8))]
        keep.append(bufs)
        arr[j].cam = _cam(s["calib"])
        arr[j].rgb, arr[j].live_depth, arr[j].live_validity, arr[j].bg_depth, \
            arr[j].bg_validity = [_p(b) for b in bufs]
        arr[j].weight = blend_weight(s["calib"], dst, cfg["mixing_epsilon"])
    c = _Cfg(cfg["splat_radius"], cfg["crack_fill_window"], cfg["depth_band_rel"])
    c.hole_color[:] = list(cfg["hole_color"])
    rgb = np.empty((dst.height, dst.width, 3), np.uint8)
    prov = np.empty((dst.height, dst.width), np.uint8)
    if lib().fo_synthesize_view(C.byref(_cam(virtual)), arr, len(refs), C.byref(c), _p(rgb),
                                _p(prov)):
        raise ValueError("fo_synthesize_view failed")
    return rgb, prov


def es_view(virtual, frames, cfg=None, hole_closing=True):
    refs = []
    for f in frames:
        d, v = decode_mm(f["mm"], f["validity"])
        if hole_closing:
            d, v = bilateral_close_holes(d, v, f["rgb"])
        refs.append(dict(calib=f["calib"], rgb=f["rgb"], live_depth=d, live_validity=v,
                         bg_depth=f["bg_depth"], bg_validity=f["bg_validity"]))
    return synthesize_view(virtual, refs, cfg)

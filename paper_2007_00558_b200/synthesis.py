"""Layered DIBR view synthesis on B200 — drop-in for ``fvv.synthesis``.

Same public names, signatures, return types and ``ValueError`` cases as the
reference module (``/root/reference/pkg/src/fvv/synthesis.py``); every raster
operation runs in the sm_100a kernels of ``libfvvb200.so`` through the C ABI
(``include/fvv_b200.h``):

=======================  ==============================  =====================
this module              reference                       C ABI / kernels
=======================  ==============================  =====================
``synthesize_view``      synthesis.py:331-362            fvv_synthesize_view (K2+K3)
``synthesize_view_debug``synthesis.py:376-397            fvv_synthesize_view + fvv_debug
``warp_layer``           synthesis.py:162-258            fvv_warp_layer
``mix_layer``            synthesis.py:261-292            fvv_mix_layer
``composite``            synthesis.py:295-318            fvv_composite
``view_psnr``            synthesis.py:439-460            host metric (not on the path)
``border_mask``          synthesis.py:463-471            host helper
=======================  ==============================  =====================

Inputs may be numpy arrays (copied to the device) or CUDA tensors; outputs
are host numpy arrays, like the reference's. There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Mapping, Optional, Sequence, Tuple

import numpy as np

from . import _dev, _native
from .geometry import camera_distance
from .types import ColorFrame, Validity

LAYER_FG = "fg"
LAYER_BG = "bg"


@dataclass(frozen=True)
class SynthesisConfig:
    """synthesis.SynthesisConfig (synthesis.py:36-49)."""

    reference_count: int = 3
    splat_radius: int = 1
    crack_fill_window: int = 3
    mixing_epsilon: float = 0.01
    depth_band_rel: float = 0.02
    hole_color: Tuple[int, int, int] = (0, 0, 0)
    # Extensions outside the reference, off by
    # default so the defaults compute exactly what the reference computes:
    #   angular_weight: blend weight 1/(dist + eps) x 1/(theta + angular_epsilon)
    #     per pixel, theta the angle at the surface point between the reference
    #     and virtual camera rays;
    #   inpaint: background-biased fill of disocclusion holes (kernel K4);
    #     provenance 3 marks inpainted pixels.
    angular_weight: bool = False
    angular_epsilon: float = 0.017453292519943295
    inpaint: bool = False
    inpaint_radius: int = 64

    def __post_init__(self):
        if self.reference_count < 1:
            raise ValueError("reference count must be >= 1")
        if self.splat_radius < 0 or self.crack_fill_window < 1:
            raise ValueError("bad splat/crack parameters")
        if self.angular_weight and not self.angular_epsilon > 0:
            raise ValueError("angular_epsilon must be positive")
        if self.inpaint and not 1 <= self.inpaint_radius <= 4096:
            raise ValueError("inpaint_radius must be in [1, 4096]")


@dataclass(frozen=True)
class LayerContribution:
    """One camera's warped layer in virtual-view coordinates (synthesis.py:52-65).

    ``winner`` / ``stage`` are extra rasters the reference does not keep:
    the z-buffer winner's source pixel index and how the pixel was covered
    (0 none, 1 centre, 2 splat, 3 crack median).
    """

    layer: str
    camera_id: int
    color: np.ndarray
    depth: np.ndarray
    valid: np.ndarray
    weight: float
    winner: Optional[np.ndarray] = field(default=None, compare=False, repr=False)
    stage: Optional[np.ndarray] = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        if self.weight <= 0:
            raise ValueError("contribution weight must be positive")


@dataclass(frozen=True)
class MergedLayer:
    color: np.ndarray
    depth: np.ndarray
    valid: np.ndarray


@dataclass(frozen=True)
class CameraStreamInputs:
    """Everything one reference camera contributes (synthesis.py:321-328)."""

    calib: object
    live_color: object
    live_depth: object
    bg_depth: object


@dataclass(frozen=True)
class DebugBundle:
    fg_contributions: Tuple[LayerContribution, ...]
    bg_contributions: Tuple[LayerContribution, ...]
    fg: MergedLayer
    bg: MergedLayer
    provenance: np.ndarray


def _wh(calib):
    k = calib.intrinsics
    return int(k.width), int(k.height)


def _check_calib(calib, height, width, what="raster"):
    """A raster must have the size its calibration declares: the kernels
    read/write the calibration's W*H pixels (the reference fails in numpy
    broadcasting there)."""
    W, H = _wh(calib)
    if (int(height), int(width)) != (H, W):
        raise ValueError(f"camera {calib.id}: {what} is {width}x{height}, its intrinsics "
                         f"say {W}x{H}")


def _weight(src_calib, dst_calib, cfg) -> float:
    return 1.0 / (camera_distance(src_calib.pose, dst_calib.pose) + cfg.mixing_epsilon)


def warp_layer(color, depth, src, dst, cfg: SynthesisConfig,
               color_valid: Optional[np.ndarray] = None,
               layer: str = LAYER_FG) -> LayerContribution:
    """Warp one camera's layer into ``dst`` (synthesis.py:162-258)."""
    if (color.height, color.width) != (depth.height, depth.width):
        raise ValueError("color and depth dimensions differ")
    _check_calib(src, color.height, color.width)
    if color_valid is not None and np.shape(color_valid) != (color.height, color.width):
        raise ValueError("color_valid does not match the colour raster")
    ctx = _native.context()
    W, H = _wh(dst)
    rgb = _dev.upload(color.pixels, np.uint8)
    d = _dev.upload(depth.depth, np.float32)
    v = _dev.upload(depth.validity, np.uint8)
    cv = None if color_valid is None else _dev.upload(np.asarray(color_valid, bool), np.uint8)
    out_c = _dev.empty((H, W, 3), np.float64)
    out_d = _dev.empty((H, W), np.float64)
    out_v = _dev.empty((H, W), np.uint8)
    out_w = _dev.empty((H, W), np.int32)
    out_s = _dev.empty((H, W), np.uint8)
    ctx.call("fvv_warp_layer", C.byref(_native.camera(src)), C.byref(_native.camera(dst)),
             rgb.data_ptr(), d.data_ptr(), v.data_ptr(), _dev.ptr(cv),
             1 if layer == LAYER_FG else 0, C.byref(_native.synth_cfg(cfg)),
             out_c.data_ptr(), out_d.data_ptr(), out_v.data_ptr(), out_w.data_ptr(),
             out_s.data_ptr())
    return LayerContribution(layer=layer, camera_id=src.id, color=_dev.host(out_c),
                             depth=_dev.host(out_d), valid=_dev.host(out_v).astype(bool),
                             weight=_weight(src, dst, cfg), winner=_dev.host(out_w),
                             stage=_dev.host(out_s))


def mix_layer(contribs: Sequence[LayerContribution], cfg: SynthesisConfig) -> MergedLayer:
    """Distance-weighted blend within the depth band (synthesis.py:261-292)."""
    if not contribs:
        raise ValueError("need at least one contribution")
    ctx = _native.context()
    H, W = np.asarray(contribs[0].valid).shape
    for c in contribs:
        if np.shape(c.valid) != (H, W) or np.shape(c.depth) != (H, W) or \
                np.shape(c.color) != (H, W, 3):
            raise ValueError("contribution dimensions differ")
    cols = [_dev.upload(c.color, np.float64) for c in contribs]
    deps = [_dev.upload(c.depth, np.float64) for c in contribs]
    vals = [_dev.upload(np.asarray(c.valid, bool), np.uint8) for c in contribs]
    n = len(contribs)
    arr = C.c_void_p * n
    wts = (C.c_double * n)(*[float(c.weight) for c in contribs])
    out_c = _dev.empty((H, W, 3), np.float64)
    out_d = _dev.empty((H, W), np.float64)
    out_v = _dev.empty((H, W), np.uint8)
    ctx.call("fvv_mix_layer", n, arr(*[t.data_ptr() for t in cols]),
             arr(*[t.data_ptr() for t in deps]), arr(*[t.data_ptr() for t in vals]), wts, W, H,
             float(cfg.depth_band_rel), out_c.data_ptr(), out_d.data_ptr(), out_v.data_ptr())
    return MergedLayer(color=_dev.host(out_c), depth=_dev.host(out_d),
                       valid=_dev.host(out_v).astype(bool))


def composite(fg: MergedLayer, bg: MergedLayer, cfg: SynthesisConfig,
              return_provenance: bool = False):
    """FG over BG over hole colour; provenance 0 hole / 1 bg / 2 fg (synthesis.py:295-318)."""
    if np.asarray(fg.valid).shape != np.asarray(bg.valid).shape:
        raise ValueError("layer dimensions differ")
    shape = np.asarray(fg.valid).shape
    if np.shape(fg.color) != shape + (3,) or np.shape(bg.color) != shape + (3,):
        raise ValueError("layer dimensions differ")
    ctx = _native.context()
    H, W = np.asarray(fg.valid).shape
    fc = _dev.upload(fg.color, np.float64)
    fv = _dev.upload(np.asarray(fg.valid, bool), np.uint8)
    bc = _dev.upload(bg.color, np.float64)
    bv = _dev.upload(np.asarray(bg.valid, bool), np.uint8)
    rgb = _dev.empty((H, W, 3), np.uint8)
    prov = _dev.empty((H, W), np.uint8)
    hole = (C.c_uint8 * 3)(*[int(x) for x in cfg.hole_color])
    ctx.call("fvv_composite", fc.data_ptr(), fv.data_ptr(), bc.data_ptr(), bv.data_ptr(), W, H,
             hole, rgb.data_ptr(), prov.data_ptr())
    frame = ColorFrame(W, H, _dev.host(rgb))
    return (frame, _dev.host(prov)) if return_provenance else frame


def _ref_frames(virtual, inputs, refs, cfg):
    if not refs:
        raise ValueError("need at least one reference camera")
    if len(refs) > _native.MAX_REFS:
        raise ValueError(f"at most {_native.MAX_REFS} reference cameras")
    frames = (_native.FvvRefFrame * len(refs))()
    keep = []
    for j, rid in enumerate(refs):
        if rid not in inputs:
            raise ValueError(f"missing inputs for reference camera {rid}")
        s = inputs[rid]
        for d in (s.live_depth, s.bg_depth):
            if (s.live_color.height, s.live_color.width) != (d.height, d.width):
                raise ValueError("color and depth dimensions differ")
        _check_calib(s.calib, s.live_color.height, s.live_color.width)
        bufs = (_dev.upload(s.live_color.pixels, np.uint8),
                _dev.upload(s.live_depth.depth, np.float32),
                _dev.upload(s.live_depth.validity, np.uint8),
                _dev.upload(s.bg_depth.depth, np.float32),
                _dev.upload(s.bg_depth.validity, np.uint8))
        keep.append(bufs)
        f = frames[j]
        f.cam = _native.camera(s.calib)
        f.rgb, f.live_depth, f.live_validity, f.bg_depth, f.bg_validity = \
            [b.data_ptr() for b in bufs]
        f.weight = _weight(s.calib, virtual, cfg)
    return frames, keep


def synthesize_view(virtual, inputs: Mapping[int, CameraStreamInputs], refs: Sequence[int],
                    cfg: SynthesisConfig, return_provenance: bool = False):
    """Render ``virtual`` from ``refs`` (synthesis.py:331-362) on the GPU."""
    frames, _keep = _ref_frames(virtual, inputs, refs, cfg)
    ctx = _native.context()
    W, H = _wh(virtual)
    rgb = _dev.empty((H, W, 3), np.uint8)
    prov = _dev.empty((H, W), np.uint8) if return_provenance else None
    ctx.call("fvv_synthesize_view", C.byref(_native.camera(virtual)), frames, len(refs),
             C.byref(_native.synth_cfg(cfg)), rgb.data_ptr(), _dev.ptr(prov), None)
    frame = ColorFrame(W, H, _dev.host(rgb))
    return (frame, _dev.host(prov)) if return_provenance else frame


def synthesize_view_debug(virtual, inputs: Mapping[int, CameraStreamInputs],
                          refs: Sequence[int], cfg: SynthesisConfig):
    """synthesize_view plus every intermediate raster (synthesis.py:376-397)."""
    frames, _keep = _ref_frames(virtual, inputs, refs, cfg)
    ctx = _native.context()
    W, H = _wh(virtual)
    n = len(refs)
    rgb = _dev.empty((H, W, 3), np.uint8)
    prov = _dev.empty((H, W), np.uint8)
    cc = _dev.empty((2 * n, H, W, 3), np.float64)
    cd = _dev.empty((2 * n, H, W), np.float64)
    cv = _dev.empty((2 * n, H, W), np.uint8)
    cw = _dev.empty((2 * n, H, W), np.int32)
    cs = _dev.empty((2 * n, H, W), np.uint8)
    mc = _dev.empty((2, H, W, 3), np.float64)
    md = _dev.empty((2, H, W), np.float64)
    mv = _dev.empty((2, H, W), np.uint8)
    dbg = _native.FvvDebug(*[t.data_ptr() for t in (cc, cd, cv, cw, cs, mc, md, mv)])
    ctx.call("fvv_synthesize_view", C.byref(_native.camera(virtual)), frames, n,
             C.byref(_native.synth_cfg(cfg)), rgb.data_ptr(), prov.data_ptr(), C.byref(dbg))
    rgb, prov, cc, cd, cv, cw, cs, mc, md, mv = [
        _dev.host(t) for t in (rgb, prov, cc, cd, cv, cw, cs, mc, md, mv)]
    contribs = []
    for k in range(2 * n):
        rid = refs[k % n]
        s = inputs[rid]
        layer = LAYER_FG if k < n else LAYER_BG
        contribs.append(LayerContribution(layer, s.calib.id, cc[k], cd[k], cv[k].astype(bool),
                                          frames[k % n].weight, cw[k], cs[k]))
    fg = MergedLayer(mc[0], md[0], mv[0].astype(bool))
    bg = MergedLayer(mc[1], md[1], mv[1].astype(bool))
    frame = ColorFrame(W, H, rgb)
    return frame, DebugBundle(tuple(contribs[:n]), tuple(contribs[n:]), fg, bg, prov)


def _rounded_rgb(color: np.ndarray) -> np.ndarray:
    """np.clip(np.round(color), 0, 255).astype(uint8) (synthesis.py:419) on the
    device: the composite kernel's half-even saturating conversion with the
    layer valid everywhere."""
    H, W = color.shape[:2]
    ones = np.ones((H, W), bool)
    fg = MergedLayer(np.asarray(color, np.float64), np.zeros((H, W)), ones)
    return composite(fg, fg, SynthesisConfig()).pixels


def write_debug_bundle(root, frame_id: int, bundle: DebugBundle, timestamp_us: int = 0) -> None:
    """Debug-raster dump in the MVD container layout (synthesis.py:400-436):
    each layer's contributions in ``<root>/<layer>/`` keyed by source camera,
    the merged layer in the reserved virtual camera slot 15, the provenance
    map as an 8-bit PNG. Written with this package's ``mvdio.MvdWriter``
    (mm quantisation and validity run-length code on the GPU)."""
    from pathlib import Path

    from PIL import Image

    from .mvdio import MvdWriter
    from .types import DepthFrame, MvdFrame

    root = Path(root)

    def to_frame(camera_id, color, depth, valid):
        valid = np.asarray(valid, bool)
        h, w = valid.shape
        validity = np.where(valid, Validity.VALID, Validity.INVALID).astype(np.uint8)
        d = np.where(valid, depth, 0.0).astype(np.float32)
        return MvdFrame(camera_id=camera_id, color=ColorFrame(w, h, _rounded_rgb(color),
                                                              timestamp_us),
                        depth=DepthFrame(w, h, d, validity, timestamp_us))

    for layer_name, contribs, merged in (("fg", bundle.fg_contributions, bundle.fg),
                                         ("bg", bundle.bg_contributions, bundle.bg)):
        h, w = np.asarray(merged.valid).shape
        with MvdWriter(root / layer_name, 0.0, w, h) as writer:
            for c in contribs:
                writer.write_frame(frame_id, to_frame(c.camera_id, c.color, c.depth, c.valid))
            writer.write_frame(frame_id, to_frame(15, merged.color, merged.depth, merged.valid))
    Image.fromarray(np.asarray(bundle.provenance, np.uint8), mode="L").save(
        root / f"{frame_id:06d}.provenance.png")


def view_psnr(synth, oracle, exclude: Optional[np.ndarray] = None) -> float:
    """Masked PSNR in dB (synthesis.py:439-460); inf for identical images."""
    if (synth.height, synth.width) != (oracle.height, oracle.width):
        raise ValueError("image dimensions differ")
    keep = np.ones((synth.height, synth.width), dtype=bool)
    if exclude is not None:
        keep &= ~np.asarray(exclude, dtype=bool)
    if not keep.any():
        raise ValueError("all pixels excluded; PSNR undefined")
    diff = synth.pixels[keep].astype(np.float64) - oracle.pixels[keep].astype(np.float64)
    mse = float(np.mean(diff ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(255.0 ** 2 / mse)


def border_mask(height: int, width: int, border: int) -> np.ndarray:
    m = np.zeros((height, width), dtype=bool)
    if border > 0:
        m[:border] = True
        m[-border:] = True
        m[:, :border] = True
        m[:, -border:] = True
    return m


__all__ = ["LAYER_FG", "LAYER_BG", "SynthesisConfig", "LayerContribution", "MergedLayer",
           "CameraStreamInputs", "DebugBundle", "warp_layer", "mix_layer", "composite",
           "synthesize_view", "synthesize_view_debug", "write_debug_bundle", "view_psnr",
           "border_mask", "Validity"]

"""ctypes binding of ``libfvvb200.so`` (the C ABI in ``include/fvv_b200.h``).

The shared library is built in-tree by ``paper_2007_00558_b200.build``. There
is no CPU fallback: if the library is missing, importing the compute modules
raises ``ImportError``; if no CUDA device is present, creating a context raises
``RuntimeError``. Status codes map to the reference's exceptions:
``FVV_EINVAL`` -> ``ValueError`` (the reference raises ValueError for every
argument error), ``FVV_ECUDA`` -> ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

import os

# FVV_B200_LIB overrides the library path (kernel-variant experiments only)
LIB_PATH = Path(os.environ.get("FVV_B200_LIB") or Path(__file__).with_name("libfvvb200.so"))

FVV_OK, FVV_EINVAL, FVV_ECUDA = 0, 1, 2
MAX_REFS = 16
MAX_SLOTS = 64
ANGULAR_EPSILON = 0.017453292519943295  # 1 degree (extension default)
INPAINT_RADIUS = 64                     # pixels (extension default)

# every entry point declared in include/fvv_b200.h
EXPORTS = (
    "fvv_ctx_create", "fvv_ctx_destroy", "fvv_ctx_set_stream", "fvv_sync", "fvv_last_error",
    "fvv_version", "fvv_launch_count", "fvv_decode_mm", "fvv_decode_yuv420_12",
    "fvv_dequantize12", "fvv_bilateral_close_holes", "fvv_synthesize_view", "fvv_warp_layer",
    "fvv_mix_layer", "fvv_composite", "fvv_slot_set_camera", "fvv_slot_set_bg",
    "fvv_slot_ingest", "fvv_slot_ingest_mm", "fvv_slot_ingest_yuv", "fvv_render_views",
    "fvv_profile_enable", "fvv_profile_read", "fvv_selftest_division",
    "fvv_correct_depth", "fvv_bg_train", "fvv_classify_fg", "fvv_remove_bg_depth",
    "fvv_quantize12", "fvv_pack_yuv420", "fvv_capture_encode", "fvv_slots_ingest_mm",
    "fvv_set_range_weights", "fvv_rice_stream_bound", "fvv_rice_encode_plane",
    "fvv_rice_decode_plane", "fvv_rice_decode_planes", "fvv_encode_mm", "fvv_rle_decode",
    "fvv_rle_encode", "fvv_slot_reset", "fvv_ctx_device_generation", "fvv_slots_ingest_yuv",
    "fvv_profile_atomics", "fvv_count_atomics", "fvv_tickq_create", "fvv_tickq_destroy",
    "fvv_tickq_submit", "fvv_tickq_replay", "fvv_tickq_wait", "fvv_tickq_fence",
    "fvv_tickq_stats",
)
KERNELS = {"preprocess": 0, "forward_warp": 1, "resolve": 2, "fill": 3, "other": 4}


class FvvCamera(C.Structure):
    _fields_ = [("id", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("reserved", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("R", C.c_double * 9),
                ("C", C.c_double * 3)]


class FvvSynthCfg(C.Structure):
    _fields_ = [("splat_radius", C.c_int32), ("crack_fill_window", C.c_int32),
                ("mixing_epsilon", C.c_double), ("depth_band_rel", C.c_double),
                ("hole_color", C.c_uint8 * 3), ("angular_weight", C.c_uint8),
                ("inpaint", C.c_uint8), ("reserved", C.c_uint8 * 3),
                ("angular_epsilon", C.c_double), ("inpaint_radius", C.c_int32),
                ("reserved2", C.c_int32)]


class FvvRefFrame(C.Structure):
    _fields_ = [("cam", FvvCamera), ("rgb", C.c_void_p), ("live_depth", C.c_void_p),
                ("live_validity", C.c_void_p), ("bg_depth", C.c_void_p),
                ("bg_validity", C.c_void_p), ("weight", C.c_double)]


class FvvDebug(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "contrib_color", "contrib_depth", "contrib_valid", "contrib_winner", "contrib_stage",
        "merged_color", "merged_depth", "merged_valid")]


_VP, _I32, _D = C.c_void_p, C.c_int32, C.c_double
_SIGS = {
    "fvv_ctx_create": ([_I32, C.POINTER(C.c_void_p)], C.c_int),
    "fvv_ctx_destroy": ([_VP], C.c_int),
    "fvv_ctx_set_stream": ([_VP, _VP], C.c_int),
    "fvv_sync": ([_VP], C.c_int),
    "fvv_last_error": ([_VP], C.c_char_p),
    "fvv_version": ([], C.c_char_p),
    "fvv_launch_count": ([_VP], C.c_int64),
    "fvv_decode_mm": ([_VP, _VP, _VP, _I32, _I32, _VP, _VP], C.c_int),
    "fvv_decode_yuv420_12": ([_VP, _VP, _VP, _VP, _I32, _I32, _D, _D, _VP, _VP, _VP], C.c_int),
    "fvv_dequantize12": ([_VP, _VP, _I32, _I32, _D, _D, _VP, _VP], C.c_int),
    "fvv_bilateral_close_holes": ([_VP, _VP, _VP, _VP, _I32, _I32, _I32, _D, _D, _I32, _VP,
                                   _VP, _VP], C.c_int),
    "fvv_synthesize_view": ([_VP, C.POINTER(FvvCamera), C.POINTER(FvvRefFrame), _I32,
                             C.POINTER(FvvSynthCfg), _VP, _VP, C.POINTER(FvvDebug)], C.c_int),
    "fvv_warp_layer": ([_VP, C.POINTER(FvvCamera), C.POINTER(FvvCamera), _VP, _VP, _VP, _VP,
                        _I32, C.POINTER(FvvSynthCfg), _VP, _VP, _VP, _VP, _VP], C.c_int),
    "fvv_mix_layer": ([_VP, _I32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                       C.POINTER(C.c_void_p), C.POINTER(C.c_double), _I32, _I32, _D, _VP, _VP,
                       _VP], C.c_int),
    "fvv_composite": ([_VP, _VP, _VP, _VP, _VP, _I32, _I32, C.POINTER(C.c_uint8), _VP, _VP],
                      C.c_int),
    "fvv_slot_set_camera": ([_VP, _I32, C.POINTER(FvvCamera)], C.c_int),
    "fvv_slot_set_bg": ([_VP, _I32, _VP, _VP], C.c_int),
    "fvv_slot_reset": ([_VP, _I32], C.c_int),
    "fvv_ctx_device_generation": ([_VP, _I32], C.c_int),
    "fvv_profile_atomics": ([_VP, C.POINTER(C.c_int64)], C.c_int),
    "fvv_count_atomics": ([_VP, _I32], C.c_int),
    "fvv_slots_ingest_yuv": ([_VP, _I32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                              C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                              C.POINTER(C.c_void_p), _D, _D, _I32], C.c_int),
    "fvv_slot_ingest": ([_VP, _I32, _VP, _VP, _VP, _I32], C.c_int),
    "fvv_slot_ingest_mm": ([_VP, _I32, _VP, _VP, _VP, _I32, _VP, _VP], C.c_int),
    "fvv_slot_ingest_yuv": ([_VP, _I32, _VP, _VP, _VP, _VP, _D, _D, _I32, _VP, _VP], C.c_int),
    "fvv_profile_enable": ([_VP, _I32], C.c_int),
    "fvv_selftest_division": ([_VP, C.c_int64, C.c_uint64, _I32, _VP], C.c_int),
    "fvv_profile_read": ([_VP, _I32, C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
    "fvv_correct_depth": ([_VP, _VP, _VP, _I32, _I32, _D, _D, _VP, _VP], C.c_int),
    "fvv_bg_train": ([_VP, _VP, _I32, _I32, _VP, _VP, _I32, _D, _D], C.c_int),
    "fvv_classify_fg": ([_VP, _VP, _VP, _VP, _I32, _I32, _D, _VP], C.c_int),
    "fvv_remove_bg_depth": ([_VP, _VP, _VP, _VP, _I32, _I32, _VP, _VP], C.c_int),
    "fvv_quantize12": ([_VP, _VP, _VP, _I32, _I32, _D, _D, _VP], C.c_int),
    "fvv_pack_yuv420": ([_VP, _VP, _I32, _I32, _VP, _VP, _VP], C.c_int),
    "fvv_capture_encode": ([_VP, _VP, _VP, _VP, _I32, _I32, _I32, _D, _D, _VP, _VP, _D, _D, _D,
                            _VP, _VP, _VP, _VP], C.c_int),
    "fvv_slots_ingest_mm": ([_VP, _I32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                             C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _I32], C.c_int),
    "fvv_set_range_weights": ([_VP, _D, C.POINTER(C.c_double), _I32], C.c_int),
    "fvv_rice_stream_bound": ([_I32, _I32], C.c_int64),
    "fvv_rice_encode_plane": ([_VP, _VP, _I32, _I32, _VP, C.POINTER(C.c_int32),
                               C.POINTER(C.c_int64)], C.c_int),
    "fvv_rice_decode_plane": ([_VP, _VP, C.c_int64, _I32, C.c_int64, _I32, _I32, _VP,
                               C.POINTER(C.c_uint32)], C.c_int),
    "fvv_rice_decode_planes": ([_VP, _I32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_void_p), C.POINTER(C.c_uint32),
                                C.POINTER(C.c_int32)], C.c_int),
    "fvv_encode_mm": ([_VP, _VP, _VP, _I32, _I32, _VP], C.c_int),
    "fvv_rle_decode": ([_VP, _VP, _VP, C.c_int64, C.c_int64, _VP], C.c_int),
    "fvv_rle_encode": ([_VP, _VP, C.c_int64, _VP, _VP, C.POINTER(C.c_int64)], C.c_int),
    "fvv_render_views": ([_VP, C.POINTER(FvvCamera), _I32, C.POINTER(C.c_int32),
                          C.POINTER(C.c_double), _I32, C.POINTER(FvvSynthCfg), _VP, _VP],
                         C.c_int),
    "fvv_tickq_create": ([_VP, _I32, C.c_int64, C.c_int64, _I32, C.POINTER(C.c_void_p)], C.c_int),
    "fvv_tickq_destroy": ([_VP], C.c_int),
    "fvv_tickq_submit": ([_VP, _VP, C.c_int64, _I32, _I32, C.POINTER(C.c_int32),
                          C.POINTER(C.c_int64), _D, _D, _I32, C.POINTER(FvvCamera), _I32,
                          C.POINTER(C.c_int32), C.POINTER(C.c_double), _I32,
                          C.POINTER(FvvSynthCfg), _VP, C.c_uint64, C.POINTER(C.c_int64)],
                         C.c_int),
    "fvv_tickq_replay": ([_VP, _VP, C.c_int64, _VP, C.c_uint64, C.POINTER(C.c_int64)], C.c_int),
    "fvv_tickq_wait": ([_VP, C.c_int64], C.c_int),
    "fvv_tickq_fence": ([_VP, _VP], C.c_int),
    "fvv_tickq_stats": ([_VP] + [C.POINTER(C.c_int64)] * 5, C.c_int),
}

_lib = None
_lock = threading.Lock()

# K1's range factor np.exp(-color_d2 * inv_2sr) (depthproc.py:200,211-212) takes
# its argument from a finite integer set (d2 = sum of three squared u8
# differences), so the host evaluates it once per sigma with the very np.exp
# the reference calls, and the kernel reads the table. numpy's SIMD exp and
# libm's differ in the last bit on ~5 % of these arguments.
RANGE_TABLE_LEN = 3 * 255 * 255 + 1
_DEFAULT_SIGMA_RANGE = 10.0  # depthproc.py:176
# entry points that run K1 with the reference defaults when hole_closing != 0
_DEFAULT_HOLE_CLOSING = frozenset((
    "fvv_slot_ingest", "fvv_slot_ingest_mm", "fvv_slots_ingest_mm", "fvv_slot_ingest_yuv",
    "fvv_slots_ingest_yuv"))


def range_weight_table(sigma_range: float) -> np.ndarray:
    """np.exp(-color_d2 * inv_2sr) for color_d2 = 0 .. 3*255^2, in the
    reference's own expression (depthproc.py:200,212)."""
    inv_2sr = 1.0 / (2.0 * float(sigma_range) ** 2)
    color_d2 = np.arange(RANGE_TABLE_LEN, dtype=np.float64)
    return np.ascontiguousarray(np.exp(-color_d2 * inv_2sr))


def load() -> C.CDLL:
    """Load and type the shared library; raise ImportError when it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g;"
                    f" g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
            lib = C.CDLL(str(LIB_PATH))
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
        return _lib


def camera(calib) -> FvvCamera:
    """fvv_camera from any object shaped like ``core.CameraCalibration``."""
    k = calib.intrinsics
    c = FvvCamera()
    c.id = int(calib.id)
    c.width, c.height = int(k.width), int(k.height)
    c.fx, c.fy, c.cx, c.cy = float(k.fx), float(k.fy), float(k.cx), float(k.cy)
    c.R[:] = [float(x) for x in np.asarray(calib.pose.rotation, dtype=np.float64).ravel()]
    c.C[:] = [float(x) for x in np.asarray(calib.pose.center, dtype=np.float64).ravel()]
    return c


def synth_cfg(cfg) -> FvvSynthCfg:
    s = FvvSynthCfg()
    s.splat_radius = int(cfg.splat_radius)
    s.crack_fill_window = int(cfg.crack_fill_window)
    s.mixing_epsilon = float(cfg.mixing_epsilon)
    s.depth_band_rel = float(cfg.depth_band_rel)
    s.hole_color[:] = [int(x) for x in cfg.hole_color]
    # extensions (absent from the reference's SynthesisConfig -> parity mode)
    s.angular_weight = int(bool(getattr(cfg, "angular_weight", False)))
    s.inpaint = int(bool(getattr(cfg, "inpaint", False)))
    s.angular_epsilon = float(getattr(cfg, "angular_epsilon", ANGULAR_EPSILON))
    s.inpaint_radius = int(getattr(cfg, "inpaint_radius", INPAINT_RADIUS))
    return s


class Context:
    """One library context (device + stream + resident slots and canvases)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = C.c_void_p()
        rc = self.lib.fvv_ctx_create(int(device), C.byref(h))
        if rc != FVV_OK:
            raise RuntimeError(f"fvv_ctx_create(device={device}) failed with status {rc} "
                               "(no CUDA device?)")
        self.h = h
        self.device = int(device)
        self._range_sigma = None
        self._free_slots = list(range(MAX_SLOTS))
        self.range_weights(_DEFAULT_SIGMA_RANGE)

    def alloc_slots(self, n: int):
        """Reserve ``n`` camera slots of this context (lowest free ids), or
        None when fewer than ``n`` are free. Renderers sharing a context hold
        disjoint slots, so one never renders another's frames."""
        with _lock:
            if n > len(self._free_slots):
                return None
            got, self._free_slots = self._free_slots[:n], self._free_slots[n:]
            return got

    def free_slots(self, slots) -> None:
        with _lock:
            self._free_slots = sorted(set(self._free_slots) | set(slots))

    def range_weights(self, sigma_range: float) -> None:
        """Make K1's resident range-weight table the np.exp one for sigma_range."""
        sigma_range = float(sigma_range)
        if self._range_sigma == sigma_range:
            return
        t = range_weight_table(sigma_range)
        self.check(self.lib.fvv_set_range_weights(
            self.h, sigma_range, t.ctypes.data_as(C.POINTER(C.c_double)), RANGE_TABLE_LEN),
            "fvv_set_range_weights")
        self._range_sigma = sigma_range

    def check(self, rc: int, what: str = "") -> None:
        if rc == FVV_OK:
            return
        msg = (self.lib.fvv_last_error(self.h) or b"").decode()
        if rc == FVV_EINVAL:
            raise ValueError(msg or what)
        raise RuntimeError(f"{what}: {msg}")

    def call(self, name: str, *args) -> None:
        if name in _DEFAULT_HOLE_CLOSING:
            self.range_weights(_DEFAULT_SIGMA_RANGE)
        self.check(getattr(self.lib, name)(self.h, *args), name)

    def set_stream(self, stream_handle: int) -> None:
        self.check(self.lib.fvv_ctx_set_stream(self.h, C.c_void_p(stream_handle)))

    def launches(self) -> int:
        return int(self.lib.fvv_launch_count(self.h))

    def profile(self, enable: bool) -> None:
        self.check(self.lib.fvv_profile_enable(self.h, int(bool(enable))), "profile")

    def profile_read(self) -> dict:
        out = {}
        for name, kid in KERNELS.items():
            ms, n = C.c_double(), C.c_int64()
            self.check(self.lib.fvv_profile_read(self.h, kid, C.byref(ms), C.byref(n)))
            out[name] = (ms.value, n.value)
        return out

    def count_atomics(self, enable: bool) -> None:
        """Counting pass on/off (resets): K2 counts its z-buffer atomics."""
        self.check(self.lib.fvv_count_atomics(self.h, int(bool(enable))), "count_atomics")

    def profile_atomics(self) -> int:
        """K2's z-buffer atomics counted since count_atomics(True)."""
        n = C.c_int64()
        self.check(self.lib.fvv_profile_atomics(self.h, C.byref(n)), "profile_atomics")
        return int(n.value)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.fvv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict = {}


def context(device: int | None = None) -> Context:
    """Per-device default context, bound to torch's current stream."""
    import torch

    if device is None:
        device = torch.cuda.current_device()
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = _contexts[device] = Context(device)
    ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
    return ctx

"""Edge-server session: resident camera slots and batched view rendering.

``EdgeRenderer`` is the B200 form of the reference's edge-server render tick
(``EdgeServer.render_tick``, pipeline.py:496-566): it keeps, per rig camera,
the calibration, the static background model (uploaded once, pipeline.py:445)
and the latest live frame resident in HBM; ``render`` then synthesizes any
number of virtual views from them (``synthesize_with_config`` seam,
pipeline.py:569-570). Frames arrive either as DepthFrames or in the wire
formats the edge server decodes (16-bit mm raster, 12-bit YUV420), with the
decode + ingest in one kernel (K0) for all of a tick's cameras, followed by
the hole fill (K1) of the pixels K0 listed.

``synthesize(virtual_camera, mvd_frame, ...)`` is the one-call convenience
the north star names.
"""

from __future__ import annotations

import ctypes as C
from collections import OrderedDict
from typing import Mapping, Optional, Sequence

import numpy as np
import torch

from . import _dev, _native
from .geometry import camera_distance
from .selection import select_references
from .synthesis import SynthesisConfig
from .types import ColorFrame


class EdgeRenderer:
    def __init__(self, rig: Sequence, bg_models: Optional[Mapping] = None,
                 cfg: Optional[SynthesisConfig] = None, device: Optional[int] = None,
                 private: bool = False):
        """``private=True`` gives the renderer its own library context (own
        slots, canvases and stream binding), so several renderers can work on
        different frames concurrently on different CUDA streams. The default
        shares the device's context (and its z canvases) but reserves its own
        camera slots in it, so renderers never see each other's frames; when
        the shared context has too few free slots, a private one is made.
        Renderers sharing the context also share its z canvases: use them
        from one stream at a time (or make them private)."""
        self.cfg = cfg or SynthesisConfig()
        self.rig = list(rig)
        self.by_id = {c.id: c for c in self.rig}
        if len(self.by_id) != len(self.rig):
            raise ValueError("camera ids of the rig must be unique")
        if len(self.rig) > _native.MAX_SLOTS:
            raise ValueError(f"at most {_native.MAX_SLOTS} cameras per renderer")
        dev = torch.cuda.current_device() if device is None else device
        slots = None
        if not private:
            self.ctx = _native.context(dev)
            slots = self.ctx.alloc_slots(len(self.rig))
        if slots is None:
            self.ctx = _native.Context(dev)
            slots = self.ctx.alloc_slots(len(self.rig))
        self._slots = slots
        self.slot = {c.id: s for c, s in zip(self.rig, slots)}
        for c in self.rig:
            self.ctx.call("fvv_slot_set_camera", self.slot[c.id], C.byref(_native.camera(c)))
            self.ctx.call("fvv_slot_reset", self.slot[c.id])
        self.ingested = set()
        for cid, bg in (bg_models or {}).items():
            self.set_bg_model(cid, bg)

    def close(self) -> None:
        """Give the renderer's camera slots back to its context."""
        slots, self._slots = getattr(self, "_slots", None), None
        if slots:
            self.ctx.free_slots(slots)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- argument checks (the kernels read/write W*H elements of the slot's
    # calibration: a short raster must fail here, as ValueError, like the
    # reference's frame validation, core.py:96-126)

    def _hw(self, cid):
        k = self.by_id[cid].intrinsics
        return int(k.height), int(k.width)

    def _check(self, a, cid, what: str, channels: Optional[int] = None):
        H, W = self._hw(cid)
        shape = (H, W) if channels is None else (H, W, channels)
        got = tuple(getattr(a, "shape", np.shape(a)))
        if got != shape:
            raise ValueError(f"camera {cid}: {what} has shape {got}, its calibration needs {shape}")
        return a

    def _bind(self):
        self.ctx.set_stream(torch.cuda.current_stream(self.ctx.device).cuda_stream)

    def _slot(self, cid) -> int:
        if cid not in self.slot:
            raise ValueError(f"camera {cid} is not in the rig")
        return self.slot[cid]

    # -- per-session / per-frame inputs --------------------------------------

    def set_bg_model(self, cid, depth, validity=None) -> None:
        """Static background depth model of camera ``cid`` (DepthFrame or arrays)."""
        self._bind()
        self._slot(cid)
        if validity is None:
            depth, validity = depth.depth, depth.validity
        self._check(depth, cid, "background depth")
        self._check(validity, cid, "background validity")
        d = _dev.upload(depth, np.float32)
        v = _dev.upload(validity, np.uint8)
        self.ctx.call("fvv_slot_set_bg", self._slot(cid), d.data_ptr(), v.data_ptr())

    def ingest(self, cid, color, depth, hole_closing: bool = True) -> None:
        """Live ColorFrame + DepthFrame of camera ``cid`` (pipeline.py:514-524)."""
        self._bind()
        self._slot(cid)
        self._check(getattr(color, "pixels", color), cid, "colour", 3)
        self._check(depth.depth, cid, "depth")
        self._check(depth.validity, cid, "validity")
        rgb = _dev.upload(getattr(color, "pixels", color), np.uint8)
        d = _dev.upload(depth.depth, np.float32)
        v = _dev.upload(depth.validity, np.uint8)
        self.ctx.call("fvv_slot_ingest", self._slot(cid), rgb.data_ptr(), d.data_ptr(),
                      v.data_ptr(), int(bool(hole_closing)))
        self.ingested.add(cid)

    def ingest_mm(self, cid, rgb, mm, validity, hole_closing: bool = True,
                  depth_out: Optional[torch.Tensor] = None,
                  validity_out: Optional[torch.Tensor] = None) -> None:
        """Live frame as the 16-bit mm raster + validity sidecar (mvdio.py:132):
        mm decode + ingest (K0), then the bilateral hole fill (K1)."""
        self._bind()
        self._slot(cid)
        self._check(rgb, cid, "colour", 3)
        self._check(mm, cid, "mm raster")
        if validity is not None:
            self._check(validity, cid, "validity")
        for o, what in ((depth_out, "depth_out"), (validity_out, "validity_out")):
            if o is not None:
                self._check(o, cid, what)
                _dev.check_out(o, torch.float32 if what == "depth_out" else torch.uint8, what,
                               dev=self.ctx.device)
        rgb_t = _dev.upload(rgb, np.uint8)
        mm_t = _dev.upload(mm, np.uint16)
        v_t = None if validity is None else _dev.upload(validity, np.uint8)
        self.ctx.call("fvv_slot_ingest_mm", self._slot(cid), rgb_t.data_ptr(), mm_t.data_ptr(),
                      _dev.ptr(v_t), int(bool(hole_closing)), _dev.ptr(depth_out),
                      _dev.ptr(validity_out))
        self.ingested.add(cid)

    def ingest_mm_many(self, frames: Mapping, hole_closing: bool = True) -> None:
        """``{cam_id: (rgb, mm, validity)}`` in one K0 launch (one grid layer
        per camera) — the form a render tick uses for its reference cameras."""
        self._bind()
        items = list(frames.items())
        n = len(items)
        if n > _native.MAX_REFS:
            for i in range(0, n, _native.MAX_REFS):
                self.ingest_mm_many(dict(items[i:i + _native.MAX_REFS]), hole_closing)
            return
        keep = []
        for cid, (rgb, mm, val) in items:
            self._slot(cid)
            self._check(rgb, cid, "colour", 3)
            self._check(mm, cid, "mm raster")
            if val is not None:
                self._check(val, cid, "validity")
            keep.append((_dev.upload(rgb, np.uint8), _dev.upload(mm, np.uint16),
                         None if val is None else _dev.upload(val, np.uint8)))
        arr = C.c_void_p * n
        slots = (C.c_int32 * n)(*[self._slot(cid) for cid, _ in items])
        vals = None if any(k[2] is None for k in keep) else arr(*[k[2].data_ptr() for k in keep])
        self.ctx.call("fvv_slots_ingest_mm", n, slots, arr(*[k[0].data_ptr() for k in keep]),
                      arr(*[k[1].data_ptr() for k in keep]), vals, int(bool(hole_closing)))
        self.ingested.update(cid for cid, _ in items)

    def ingest_yuv(self, cid, rgb, y, u, v, depth_range, hole_closing: bool = True) -> None:
        """Live frame as the 12-bit YUV420 depth raster (pipeline.py:469-472)."""
        self._bind()
        self._slot(cid)
        H, W = self._hw(cid)
        self._check(rgb, cid, "colour", 3)
        self._check(y, cid, "Y plane")
        for a, what in ((u, "U plane"), (v, "V plane")):
            if tuple(np.shape(a) if not hasattr(a, "shape") else a.shape) != (H // 2, W // 2):
                raise ValueError(f"camera {cid}: {what} has shape {tuple(a.shape)}, its "
                                 f"calibration needs {(H // 2, W // 2)}")
        t = [_dev.upload(a, np.uint8) for a in (rgb, y, u, v)]
        self.ctx.call("fvv_slot_ingest_yuv", self._slot(cid), *[x.data_ptr() for x in t],
                      float(depth_range.z_near), float(depth_range.z_far),
                      int(bool(hole_closing)), None, None)
        self.ingested.add(cid)

    def ingest_yuv_many(self, frames: Mapping, depth_range, hole_closing: bool = True) -> None:
        """``{cam_id: (rgb, y, u, v)}``, 12-bit YUV420 depth (pipeline.py:469-472),
        in one K0 launch (one grid layer per camera) + one K1 — a render
        tick's reference cameras in the edge server's wire format."""
        self._bind()
        items = list(frames.items())
        n = len(items)
        if n > _native.MAX_REFS:
            for i in range(0, n, _native.MAX_REFS):
                self.ingest_yuv_many(dict(items[i:i + _native.MAX_REFS]), depth_range,
                                     hole_closing)
            return
        keep = []
        for cid, (rgb, y, u, v) in items:
            self._slot(cid)
            H, W = self._hw(cid)
            self._check(rgb, cid, "colour", 3)
            self._check(y, cid, "Y plane")
            for a, what in ((u, "U plane"), (v, "V plane")):
                if tuple(a.shape) != (H // 2, W // 2):
                    raise ValueError(f"camera {cid}: {what} has shape {tuple(a.shape)}, its "
                                     f"calibration needs {(H // 2, W // 2)}")
            keep.append(tuple(_dev.upload(a, np.uint8) for a in (rgb, y, u, v)))
        arr = C.c_void_p * n
        slots = (C.c_int32 * n)(*[self._slot(cid) for cid, _ in items])
        self.ctx.call("fvv_slots_ingest_yuv", n, slots,
                      *[arr(*[k[q].data_ptr() for k in keep]) for q in range(4)],
                      float(depth_range.z_near), float(depth_range.z_far), int(bool(hole_closing)))
        self.ingested.update(cid for cid, _ in items)

    def ingest_encoded_many(self, frames: Mapping, depth_range,
                            hole_closing: bool = True) -> None:
        """Live frames in the edge server's wire format, ``{cam_id: (rgb,
        EncodedFrame)}`` with MED + Rice coded 12-bit YUV420 depth
        (pipeline.py:466-472): every camera's depth planes are decoded in one
        batched GPU call, then K0 (YUV420 decode + fill candidates) and K1."""
        from .depthcodec import decode_lossless_many

        items = list(frames.items())
        planes = decode_lossless_many([enc for _, (_, enc) in items])
        for (cid, (rgb, _)), (y, u, v) in zip(items, planes):
            self.ingest_yuv(cid, rgb, y, u, v, depth_range, hole_closing=hole_closing)

    # -- rendering -------------------------------------------------------------

    def plan(self, virtuals: Sequence, refs=None):
        """Reference ids per view (select_references over the ingested set when
        ``refs`` is None, transport.py:226-238) and the blend weights."""
        k = self.cfg.reference_count
        if refs is None:
            active = sorted(self.ingested)
            refs = [select_references(v.pose, self.rig, active, min(k, len(active)))
                    for v in virtuals]
        refs = [list(r) for r in refs]
        if not refs or any(len(r) != len(refs[0]) for r in refs):
            raise ValueError("every view of a batch needs the same number of references")
        if len(refs[0]) == 0:
            raise ValueError("need at least one reference camera")
        for r in refs:
            for cid in r:
                if cid not in self.ingested:
                    raise ValueError(f"missing inputs for reference camera {cid}")
        weights = [[1.0 / (camera_distance(self.by_id[cid].pose, v.pose) + self.cfg.mixing_epsilon)
                    for cid in r] for v, r in zip(virtuals, refs)]
        return refs, weights

    def render(self, virtuals: Sequence, refs=None, out: Optional[torch.Tensor] = None,
               provenance: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Synthesize ``len(virtuals)`` views; returns a (n, H, W, 3) uint8 CUDA tensor."""
        self._bind()
        virtuals = list(virtuals)
        refs, weights = self.plan(virtuals, refs)
        n, k = len(virtuals), len(refs[0])
        W, H = int(virtuals[0].intrinsics.width), int(virtuals[0].intrinsics.height)
        if any((int(v.intrinsics.width), int(v.intrinsics.height)) != (W, H) for v in virtuals):
            raise ValueError("every view of a batch needs the same image size")
        if out is None:
            out = _dev.empty((n, H, W, 3), np.uint8)
        else:
            _dev.check_out(out, torch.uint8, "out", (n, H, W, 3), self.ctx.device)
        if provenance is not None:
            _dev.check_out(provenance, torch.uint8, "provenance", (n, H, W), self.ctx.device)
        cams = (_native.FvvCamera * n)(*[_native.camera(v) for v in virtuals])
        slots = (C.c_int32 * (n * k))(*[self.slot[c] for r in refs for c in r])
        wts = (C.c_double * (n * k))(*[w for ws in weights for w in ws])
        self.ctx.call("fvv_render_views", cams, n, slots, wts, k,
                      C.byref(_native.synth_cfg(self.cfg)), out.data_ptr(), _dev.ptr(provenance))
        return out

    def capture_step(self, frame: Mapping, virtuals: Sequence, refs=None,
                     out: Optional[torch.Tensor] = None,
                     provenance: Optional[torch.Tensor] = None,
                     hole_closing: bool = True, depth_range=None) -> "StepGraph":
        """One render tick — ``ingest_mm_many(frame)`` (K0 + K1; with
        ``depth_range``, ``ingest_yuv_many(frame, depth_range)``) and
        ``render(virtuals, refs)`` (K2 + K3) — captured once as a CUDA graph:
        ``replay()`` re-runs the tick with one launch call, on whatever the
        device buffers of ``frame`` (and the context's slots) hold by then.
        The renderer's context switches to device-resident canvas generations
        (``fvv_ctx_device_generation``), so replays stay correct. The tick is
        run once eagerly first (allocations), which renders ``out``."""
        self._bind()
        self.ctx.call("fvv_ctx_device_generation", 1)
        virtuals = list(virtuals)
        k = virtuals[0].intrinsics
        n, H, W = len(virtuals), int(k.height), int(k.width)
        if out is None:
            out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=self.ctx.device)
        cur = torch.cuda.current_stream(self.ctx.device)

        def tick():
            if depth_range is None:
                self.ingest_mm_many(frame, hole_closing=hole_closing)
            else:
                self.ingest_yuv_many(frame, depth_range, hole_closing=hole_closing)
            self.render(virtuals, refs, out=out, provenance=provenance)

        tick()
        side = torch.cuda.Stream(self.ctx.device)
        side.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        l0 = self.ctx.launches()
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            tick()
        cur.wait_stream(side)
        self._bind()
        sg = StepGraph(self, g, out, frame)
        sg.launches = self.ctx.launches() - l0    # kernels per replay
        return sg

    def synthesize(self, virtual, mvd_frame: Optional[Mapping] = None, refs=None,
                   hole_closing: bool = True) -> ColorFrame:
        """One view on the host: optional new frame (``{id: MvdFrame}``), then render."""
        for cid, f in (mvd_frame or {}).items():
            self.ingest(cid, f.color, f.depth, hole_closing=hole_closing)
        img = self.render([virtual], None if refs is None else [refs])
        W, H = int(virtual.intrinsics.width), int(virtual.intrinsics.height)
        return ColorFrame(W, H, img[0].cpu().numpy())


class StepGraph:
    """A captured render tick (``EdgeRenderer.capture_step``): ``replay()``
    launches the whole K0 -> K1 -> K2 -> K3 sequence as one CUDA graph on
    the current stream; ``out`` receives the views."""

    def __init__(self, renderer, graph, out, frame):
        self.renderer, self.graph, self.out = renderer, graph, out
        self._keep = frame           # the device buffers the graph reads
        self.launches = None

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.out


_SESSION: list = []   # [(key, pinned objects, renderer)] of the last synthesize() call


def _session_key(rig, bg_models, cfg):
    cams = tuple((c.id, bytes(_native.camera(c))) for c in rig)
    return cams, tuple((cid, id(bg)) for cid, bg in sorted(bg_models.items())), cfg


def synthesize(virtual_camera, mvd_frame: Mapping, refs=None, cfg: Optional[SynthesisConfig] = None,
               *, rig: Sequence, bg_models: Mapping, hole_closing: bool = True) -> ColorFrame:
    """North-star convenience call: ``mvd_frame`` maps camera id -> MvdFrame;
    ``refs=None`` selects ``cfg.reference_count`` nearest cameras.

    Consecutive calls with the same rig, the same BG-model objects and the
    same config reuse one session (resident slots, BG models uploaded once,
    pipeline.py:445); the held BG objects keep their ids from being reused."""
    cfg = cfg or SynthesisConfig()
    key = _session_key(rig, bg_models, cfg)
    if _SESSION and _SESSION[0][0] == key:
        r = _SESSION[0][2]
    else:
        if _SESSION:
            _SESSION.pop()[2].close()
        r = EdgeRenderer(rig, bg_models, cfg)
        _SESSION.append((key, (list(rig), dict(bg_models)), r))
    r.ingested = set()
    return r.synthesize(virtual_camera, mvd_frame, refs, hole_closing=hole_closing)


class FrameUploader:
    """Double-buffered host->device staging of live frames on a copy stream.

    ``put(frame)`` enqueues the pinned-host -> HBM copies of one frame
    (``{cam_id: (rgb u8 HxWx3, mm int16/uint16 HxW, validity u8 HxW)}``) on a
    dedicated stream and returns a ticket; ``get(ticket)`` makes the current
    (compute) stream wait for those copies and returns the device tensors;
    ``release(ticket)`` marks the point on the compute stream after which the
    buffers may be overwritten by the copy ``depth`` puts later.
    With ``depth`` >= 2 the upload of frame t+1 overlaps the synthesis of
    frame t, so a PCIe-fed edge server is bounded by the link, not by
    copy + compute in series.
    """

    def __init__(self, example_frame: Mapping, depth: int = 2, device=None, lanes: int = None):
        self.dev = _dev.device() if device is None else torch.device(device)
        self.stream = torch.cuda.Stream(self.dev)
        # copies spread over `lanes` streams so one copy's setup overlaps
        # another's transfer: two for frames of 8 MB and more (c1: +2 % e2e),
        # one below, where the extra events cost more than they hide
        # (FVV_UPLOAD_LANES overrides)
        import os
        nbytes = sum(t.numel() * t.element_size() for ts in example_frame.values() for t in ts)
        # a frame whose rasters all live in one host allocation (the way a
        # receive buffer holds a tick's data) moves as one span instead of
        # one copy per raster (one lane: splitting the span measured no faster)
        self.layout = self._layout(example_frame)
        if self.layout is not None:
            lanes = lanes or 1
        lanes = int(os.environ.get("FVV_UPLOAD_LANES", lanes or (2 if nbytes >= 8 << 20 else 1)))
        self.extra = [torch.cuda.Stream(self.dev) for _ in range(max(lanes, 1) - 1)]
        self.depth = depth
        if self.layout is not None:
            span = self.layout[1]
            self.flat = [torch.empty(span, dtype=torch.uint8, device=self.dev)
                         for _ in range(depth)]
            self.bufs = [{cid: tuple(self._view(self.flat[d], o, t) for o, t in zip(offs, ts))
                          for (cid, ts), offs in zip(example_frame.items(), self.layout[2])}
                         for d in range(depth)]
        else:
            self.bufs = [{cid: tuple(torch.empty(tuple(t.shape), dtype=t.dtype, device=self.dev)
                                     for t in ts) for cid, ts in example_frame.items()}
                         for _ in range(depth)]
        self.done = [None] * depth        # copy-finished events
        self.free = [None] * depth        # consumer-finished events
        # event objects reused per slot (a wait is bound to the record it
        # follows, so re-recording one later is safe); saves their creation
        # on every tick
        self._done_ev = [torch.cuda.Event() for _ in range(depth)]
        self._free_ev = [torch.cuda.Event() for _ in range(depth)]
        self._lane_ev = [[torch.cuda.Event() for _ in self.extra] for _ in range(depth)]
        self.n = 0
        self.bytes = 0

    @staticmethod
    def _layout(frame: Mapping):
        """(start, span bytes, [[byte offset per raster] per camera]) when
        every raster is a contiguous view of one allocation (offsets relative
        to the lowest raster), else None."""
        ts = [t for v in frame.values() for t in v]
        if not ts or not all(isinstance(t, torch.Tensor) and t.is_contiguous() for t in ts):
            return None
        base = ts[0].untyped_storage().data_ptr()
        if any(t.untyped_storage().data_ptr() != base for t in ts):
            return None
        lo = min(t.data_ptr() for t in ts) - base
        hi = max(t.data_ptr() + t.numel() * t.element_size() for t in ts) - base
        offs = [[t.data_ptr() - base - lo for t in v] for v in frame.values()]
        return lo, hi - lo, offs

    @staticmethod
    def _view(flat, off, t):
        n = t.numel() * t.element_size()
        return flat[off:off + n].view(t.dtype).view(tuple(t.shape))

    def put(self, frame: Mapping) -> int:
        slot = self.n % self.depth
        streams = [self.stream] + self.extra
        for st in streams:
            if self.free[slot] is not None:
                st.wait_event(self.free[slot])
        lay = self._layout(frame) if self.layout is not None else None
        if lay is not None and lay[1:] == self.layout[1:]:
            # one span, split evenly over the copy lanes
            src = torch.empty(0, dtype=torch.uint8).set_(
                next(iter(frame.values()))[0].untyped_storage(), lay[0], (lay[1],), (1,))
            step = -(-lay[1] // len(streams) // 256) * 256
            for li, st in enumerate(streams):
                a, b = li * step, min((li + 1) * step, lay[1])
                if a < b:
                    with torch.cuda.stream(st):
                        self.flat[slot][a:b].copy_(src[a:b], non_blocking=True)
            self.bytes += sum(t.numel() * t.element_size() for v in frame.values() for t in v)
        else:
            pairs = [(dst, src) for cid, ts in frame.items()
                     for dst, src in zip(self.bufs[slot][cid], ts)]
            for li, st in enumerate(streams):
                with torch.cuda.stream(st):
                    for dst, src in pairs[li::len(streams)]:
                        dst.copy_(src, non_blocking=True)
            self.bytes += sum(src.numel() * src.element_size() for _, src in pairs)
        for st, ev_l in zip(self.extra, self._lane_ev[slot]):  # the ticket's event covers every lane
            ev_l.record(st)
            self.stream.wait_event(ev_l)
        ev = self._done_ev[slot]
        ev.record(self.stream)
        self.done[slot] = ev
        self.n += 1
        return self.n - 1

    def get(self, ticket: int, stream=None) -> Mapping:
        """The ticket's device buffers; ``stream`` (default: the current one)
        waits for their copies."""
        slot = ticket % self.depth
        (stream or torch.cuda.current_stream(self.dev)).wait_event(self.done[slot])
        return self.bufs[slot]

    def release(self, ticket: int, stream=None) -> None:
        """``stream`` (default: the current one) is done reading this
        ticket's buffers."""
        slot = ticket % self.depth
        ev = self._free_ev[slot]
        ev.record(stream or torch.cuda.current_stream(self.dev))
        self.free[slot] = ev


class ResultDownloader:
    """Device -> pinned-host copies of rendered views on a separate stream.

    Render into ``next_buffer()`` (the current stream first waits until the
    download that last read that device buffer is finished, so a view is
    never overwritten while it is being copied out — the displayed frame of
    pipeline.py:546-547,762-763), then ``put`` it. Host results rotate over
    ``depth`` pinned buffers: ``on_done(host_view, tag)`` is called for each
    result once its copy has finished (before its host buffer is reused, or
    at ``flush``).
    """

    def __init__(self, shape, depth: int = 2, device=None, on_done=None):
        self.dev = _dev.device() if device is None else torch.device(device)
        self.stream = torch.cuda.Stream(self.dev)
        self.host = [torch.empty(tuple(shape), dtype=torch.uint8).pin_memory()
                     for _ in range(depth)]
        self.bufs = [torch.empty(tuple(shape), dtype=torch.uint8, device=self.dev)
                     for _ in range(depth)]
        self.depth = depth
        self.n = 0
        self.bytes = 0
        self.copied = [None] * depth       # D2H of the slot's device + host buffers done
        self.pending = [None] * depth      # (host view, tag) not yet handed to on_done
        self.on_done = on_done
        # reused per slot: a slot's copy event is re-recorded only after
        # _retire has waited for its previous record
        self._ready_ev = [torch.cuda.Event() for _ in range(depth)]
        self._copied_ev = [torch.cuda.Event() for _ in range(depth)]

    def next_buffer(self, stream=None) -> torch.Tensor:
        """The device buffer the next ``put`` downloads; safe to write on
        ``stream`` (default: the current one) from now on."""
        slot = self.n % self.depth
        if self.copied[slot] is not None:
            (stream or torch.cuda.current_stream(self.dev)).wait_event(self.copied[slot])
        return self.bufs[slot]

    def _retire(self, slot) -> None:
        if self.copied[slot] is not None:
            self.copied[slot].synchronize()
        if self.pending[slot] is not None:
            view, tag = self.pending[slot]
            self.pending[slot] = None
            if self.on_done is not None:
                self.on_done(view, tag)

    def put(self, views: torch.Tensor, tag=None, stream=None) -> torch.Tensor:
        """Queue the copy of ``views`` (after the work queued so far on
        ``stream``, default the current one); returns the pinned host tensor
        it lands in (valid once the copy is done: ``on_done``, ``flush``, or
        ``depth`` puts later). ``views`` not taken from ``next_buffer()``:
        the stream waits for the copy before running anything else, so it
        cannot be overwritten early."""
        slot = self.n % self.depth
        self._retire(slot)                 # host slot about to be reused
        cur = stream or torch.cuda.current_stream(self.dev)
        ready = self._ready_ev[slot]
        ready.record(cur)
        own = views.untyped_storage().data_ptr() == self.bufs[slot].untyped_storage().data_ptr()
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(ready)
            dst = self.host[slot][:views.shape[0]]
            dst.copy_(views, non_blocking=True)
            ev = self._copied_ev[slot]
            ev.record(self.stream)
        if not own:
            views.record_stream(self.stream)
            cur.wait_event(ev)
        self.copied[slot] = ev
        self.pending[slot] = (dst, tag)
        self.bytes += views.numel()
        self.n += 1
        return dst

    def flush(self) -> None:
        """Wait for every queued download and hand the results to on_done."""
        for i in range(self.n - self.depth, self.n):
            if i >= 0:
                self._retire(i % self.depth)

    def wait_into(self, stream) -> None:
        for ev in self.copied:
            if ev is not None:
                stream.wait_event(ev)


class TickQueue:
    """The native render-tick queue (``fvv_tickq_*``, include/fvv_b200.h):
    one tick's host span -> HBM staging slot (H2D stream) -> ingest + render
    on the renderer's stream -> views -> pinned host buffer (D2H stream),
    ``depth`` ticks in flight, repeating ticks replayed from CUDA graphs —
    every per-tick stream and event operation in native code. Used by
    ``EdgeStream`` for frames held in one host allocation."""

    def __init__(self, renderer: "EdgeRenderer", depth: int, span_bytes: int, out_bytes: int,
                 max_graphs: int):
        self.ctx = renderer.ctx
        self.lib = self.ctx.lib
        h = C.c_void_p()
        self.ctx.check(self.lib.fvv_tickq_create(self.ctx.h, int(depth), int(span_bytes),
                                                 int(out_bytes), int(max_graphs), C.byref(h)),
                       "fvv_tickq_create")
        self.h = h
        self.span_bytes, self.out_bytes = int(span_bytes), int(out_bytes)
        self._t = C.c_int64()

    def replay(self, span_ptr: int, span_bytes: int, out_ptr: int, key: int) -> int:
        """The captured tick of ``key``: its ticket, or -1 (submit it)."""
        rc = self.lib.fvv_tickq_replay(self.h, span_ptr, span_bytes, out_ptr, key,
                                       C.byref(self._t))
        if rc:
            self.ctx.check(rc, "fvv_tickq_replay")
        return self._t.value

    def submit(self, *args) -> int:
        self.ctx.check(self.lib.fvv_tickq_submit(self.h, *args, C.byref(self._t)),
                       "fvv_tickq_submit")
        return self._t.value

    def wait(self, ticket: int) -> None:
        self.ctx.check(self.lib.fvv_tickq_wait(self.h, int(ticket)), "fvv_tickq_wait")

    def fence(self, stream) -> None:
        self.ctx.check(self.lib.fvv_tickq_fence(self.h, C.c_void_p(stream.cuda_stream)),
                       "fvv_tickq_fence")

    def stats(self) -> dict:
        v = [C.c_int64() for _ in range(5)]
        self.ctx.check(self.lib.fvv_tickq_stats(self.h, *[C.byref(x) for x in v]),
                       "fvv_tickq_stats")
        return dict(zip(("ticks", "h2d_bytes", "d2h_bytes", "replays", "graphs"),
                        (x.value for x in v)))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.fvv_tickq_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _view_key(v) -> tuple:
    """A virtual camera's identity for the tick key (intrinsics + pose bytes)."""
    k = v.intrinsics
    return (int(k.width), int(k.height), float(k.fx), float(k.fy), float(k.cx), float(k.cy),
            np.asarray(v.pose.rotation, dtype=np.float64).tobytes(),
            np.asarray(v.pose.center, dtype=np.float64).tobytes())


class EdgeStream:
    """The edge server fed from host memory (the e2e path of bench.py):
    frames of pinned host rasters in, rendered views in pinned host memory
    out, with the H2D copies of frame t+1 and the D2H copy of view t-1
    overlapping frame t's decode/fill/warp/resolve on the renderer's stream.

    ``submit(frame, virtuals, refs)`` runs one render tick (pipeline.py:
    514-547): upload, ingest (K0 + K1), render (K2 + K3), download. A frame is
    ``{cam_id: (rgb, mm, validity)}`` — the 16-bit mm raster + validity
    sidecar (mvdio.py:132) — or, with ``depth_range``, ``{cam_id: (rgb, y, u,
    v)}`` — the 12-bit YUV420 depth the edge server receives on the wire
    (pipeline.py:466-472). ``on_view(host_views, tag)`` receives each tick's
    views once they are in host memory (pipeline.py:762-763 ``on_display``);
    ``flush()`` drains the last ones. With ``graphs`` (default), a tick whose
    buffers, views and references repeat is replayed from a CUDA graph
    captured on its second occurrence (at most ``max_graphs`` kept, least
    recently used dropped).

    A frame whose rasters all live in one host allocation (the way a receive
    buffer holds a tick), 16-byte aligned, goes through the native tick queue
    (``TickQueue``, ``native=True``): one call per tick, its copies, events,
    ingest, render and graph replays issued in C++. Other frames go through
    ``FrameUploader`` / ``EdgeRenderer`` / ``ResultDownloader``. Either way
    the copies are asynchronous: a tick's host rasters must stay unchanged
    until its views reach ``on_view`` (or ``flush`` returns).
    """

    def __init__(self, renderer: "EdgeRenderer", max_views: int, depth: int = 2,
                 on_view=None, hole_closing: bool = True, depth_range=None,
                 graphs: bool = True, max_graphs: int = 64, native: bool = True):
        self.r = renderer
        dev = torch.device("cuda", renderer.ctx.device)
        self.dev = dev
        k = renderer.rig[0].intrinsics
        self.max_views = int(max_views)
        self._dl_shape = (max_views, int(k.height), int(k.width), 3)
        self._dl = None             # ResultDownloader of the Python path (made on first use)
        self.on_view = on_view
        self.depth = depth
        self.ups = {}
        self.hole_closing = hole_closing
        self.depth_range = depth_range
        # ticks whose key (buffer slots, cameras, references) repeats are
        # captured on their second occurrence; a moving viewer, whose every
        # tick is new, stays on host launches (no capture per tick)
        self.graphs = OrderedDict() if graphs else None
        self.seen = OrderedDict()
        self.max_graphs = max_graphs
        self.graph_launches = 0
        # native tick queue state
        self.native = native
        self.q = None
        self._qhost = None          # depth pinned host view buffers
        self._qpend = [None] * depth  # per host buffer: (ticket, views, tag)
        self._qn = 0
        self._qkeys = {}            # tick key -> id (ids never reused)
        self._qnext = 1
        self._spans = {}            # id(frame) -> (rasters, span layout)
        self._mode = None           # "native" | "python": the path of the last tick

    @property
    def dl(self) -> ResultDownloader:
        if self._dl is None:
            self._dl = ResultDownloader(self._dl_shape, self.depth, self.dev,
                                        on_done=self.on_view)
        return self._dl

    def _uploader(self, frame):
        key = tuple((cid, tuple(tuple(t.shape) for t in ts)) for cid, ts in sorted(frame.items()))
        up = self.ups.get(key)
        if up is None:
            up = self.ups[key] = FrameUploader(dict(sorted(frame.items())), self.depth, self.dev)
        return up

    @property
    def h2d_bytes(self) -> int:
        n = sum(u.bytes for u in self.ups.values())
        return n + (self.q.stats()["h2d_bytes"] if self.q is not None else 0)

    @property
    def d2h_bytes(self) -> int:
        n = self._dl.bytes if self._dl is not None else 0
        return n + (self.q.stats()["d2h_bytes"] if self.q is not None else 0)

    # -- native path ------------------------------------------------------------

    def _span(self, frame: Mapping):
        """(host pointer, span bytes, kind, camera ids, offsets, layout key) of
        a frame held in one 16-byte aligned host allocation, else None."""
        rasters = tuple(t for v in frame.values() for t in v)
        hit = self._spans.get(id(frame))
        if hit is not None and len(hit[0]) == len(rasters) and all(
                a is b for a, b in zip(hit[0], rasters)):
            return hit[1]
        per = 4 if self.depth_range is not None else 3
        ent = None
        if all(isinstance(t, torch.Tensor) and t.device.type == "cpu" for t in rasters) and \
                all(len(v) == per for v in frame.values()):
            lay = FrameUploader._layout(frame)
            if lay is not None:
                lo, span, offs = lay
                base = rasters[0].untyped_storage().data_ptr() + lo
                flat = [o for v in offs for o in (list(v) + [-1] * (4 - len(v)))]
                if base % 16 == 0 and all(o % 16 == 0 for o in flat if o >= 0):
                    cids = list(frame.keys())
                    ent = (base, span, 0 if per == 3 else 1, cids, flat,
                           (tuple(cids), tuple(flat), span))
        if len(self._spans) > 256:
            self._spans.clear()
        self._spans[id(frame)] = (rasters, ent)
        return ent

    def _retire_native(self, slot: int) -> None:
        pend, self._qpend[slot] = self._qpend[slot], None
        if pend is not None:
            self.q.wait(pend[0])
            if self.on_view is not None:
                self.on_view(pend[1], pend[2])

    def _flush_native(self) -> None:
        for i in range(self._qn - self.depth, self._qn):
            if i >= 0:
                self._retire_native(i % self.depth)

    def _submit_native(self, frame: Mapping, virtuals: Sequence, refs, tag):
        ent = self._span(frame)
        if ent is None:
            return None
        base, span, kind, cids, offs, lkey = ent
        n = len(virtuals)
        if n > self.max_views:
            raise ValueError(f"{n} views, the stream holds {self.max_views}")
        k = virtuals[0].intrinsics
        H, W = int(k.height), int(k.width)
        if self.q is None or span > self.q.span_bytes:
            if self.q is not None:
                self._flush_native()
                self.q.close()
            rk = self.r.rig[0].intrinsics
            out_bytes = self.max_views * max(H * W, int(rk.height) * int(rk.width)) * 3
            self.q = TickQueue(self.r, self.depth, span, out_bytes,
                               self.max_graphs if self.graphs is not None else 0)
            self._qhost = [torch.empty(out_bytes, dtype=torch.uint8).pin_memory()
                           for _ in range(self.depth)]
            self._qn = 0
        if self._mode == "python" and self._dl is not None:
            self._dl.flush()
        self._mode = "native"
        self.r._bind()
        slot = self._qn % self.depth
        self._retire_native(slot)
        host = self._qhost[slot]
        views = host[:n * H * W * 3].view(n, H, W, 3)
        kid = 0
        if self.graphs is not None and refs is not None:
            key = (lkey, tuple(_view_key(v) for v in virtuals), tuple(tuple(r) for r in refs),
                   self.r.cfg)
            kid = self._qkeys.get(key)
            if kid is None:
                if len(self._qkeys) >= 16 * self.max_graphs:
                    self._qkeys.clear()   # ids are never reused: stale graphs just age out
                kid = self._qkeys[key] = self._qnext
                self._qnext += 1
        l0 = self.r.ctx.launches()
        ticket = self.q.replay(base, span, host.data_ptr(), kid)
        if ticket >= 0:
            self.graph_launches += self.r.ctx.launches() - l0
        else:
            # a new tick: the renderer's raster checks and reference plan, then
            # the eager (or, on its second occurrence, capturing) submit
            for cid, ts in frame.items():
                self.r._slot(cid)
                H2, W2 = self.r._hw(cid)
                self.r._check(ts[0], cid, "colour", 3)
                self.r._check(ts[1], cid, "mm raster" if kind == 0 else "Y plane")
                if kind == 0:
                    self.r._check(ts[2], cid, "validity")
                for a, what in (((ts[2], "U plane"), (ts[3], "V plane")) if kind else ()):
                    if tuple(a.shape) != (H2 // 2, W2 // 2):
                        raise ValueError(f"camera {cid}: {what} has shape {tuple(a.shape)}, "
                                         f"its calibration needs {(H2 // 2, W2 // 2)}")
            self.r.ctx.range_weights(_native._DEFAULT_SIGMA_RANGE)
            before = set(self.r.ingested)
            self.r.ingested.update(cids)
            try:
                refs2, weights = self.r.plan(virtuals, refs)
            except ValueError:
                self.r.ingested = before
                raise
            nr = len(refs2[0])
            dr = self.depth_range
            ticket = self.q.submit(
                C.c_void_p(base), span, kind, len(cids),
                (C.c_int32 * len(cids))(*[self.r.slot[c] for c in cids]),
                (C.c_int64 * len(offs))(*offs),
                float(dr.z_near) if dr is not None else 0.0,
                float(dr.z_far) if dr is not None else 0.0, int(bool(self.hole_closing)),
                (_native.FvvCamera * n)(*[_native.camera(v) for v in virtuals]), n,
                (C.c_int32 * (n * nr))(*[self.r.slot[c] for r in refs2 for c in r]),
                (C.c_double * (n * nr))(*[w for ws in weights for w in ws]), nr,
                C.byref(_native.synth_cfg(self.r.cfg)), C.c_void_p(host.data_ptr()), kid)
        self._qpend[slot] = (ticket, views, tag)
        self._qn += 1
        return views

    # -- public ---------------------------------------------------------------------

    def submit(self, frame: Mapping, virtuals: Sequence, refs=None, tag=None) -> torch.Tensor:
        if self.native:
            got = self._submit_native(frame, virtuals, refs, tag)
            if got is not None:
                return got
        if self._mode == "native":
            self._flush_native()
        self._mode = "python"
        up = self._uploader(frame)
        ticket = up.put(dict(sorted(frame.items())))
        cur = torch.cuda.current_stream(self.dev)
        fr = up.get(ticket, cur)
        n = len(virtuals)
        out = self.dl.next_buffer(cur)[:n]
        key = None
        if self.graphs is not None and refs is not None:
            key = (id(up), ticket % up.depth, self.dl.n % self.dl.depth,
                   tuple(bytes(_native.camera(v)) for v in virtuals),
                   tuple(tuple(r) for r in refs))
        g = self.graphs.get(key) if key is not None else None
        if g is not None:
            self.graphs.move_to_end(key)
            g.replay()
            self.graph_launches += g.launches
        elif key is not None and key in self.seen:
            # a tick seen before (same buffers, views and references): capture
            # it now (its eager run renders this tick) and replay it from then on
            self.graphs[key] = self.r.capture_step(fr, virtuals, refs, out=out,
                                                   hole_closing=self.hole_closing,
                                                   depth_range=self.depth_range)
            if len(self.graphs) > self.max_graphs:
                self.graphs.popitem(last=False)
        else:
            if key is not None:
                self.seen[key] = None
                if len(self.seen) > 4 * self.max_graphs:
                    self.seen.popitem(last=False)
            if self.depth_range is None:
                self.r.ingest_mm_many(fr, hole_closing=self.hole_closing)
            else:
                self.r.ingest_yuv_many(fr, self.depth_range, hole_closing=self.hole_closing)
            self.r.render(virtuals, refs, out=out)
        up.release(ticket, cur)
        return self.dl.put(out, tag, cur)

    def wait_into(self, stream) -> None:
        """``stream`` waits (on the device) for every download queued so far."""
        if self._dl is not None:
            self._dl.wait_into(stream)
        if self.q is not None:
            self.q.fence(stream)

    def flush(self) -> None:
        if self._dl is not None:
            self._dl.flush()
        if self.q is not None:
            self._flush_native()

"""Seeded synthetic multiview-plus-depth workloads (BASELINE.json configs c0-c4).

The paper's captured ZED sequences are not available, and
the reference's own scene generator renders a different scene family (room
box + boxes/spheres, scenegen.py:293-538). This module ray-casts the scenes
BASELINE.json describes, with numpy, from a seed:

* static background = textured quads of random orientation (+ a ground plane
  for the 1080p/4K rigs); foreground = textured spheres (optionally moving);
* textures: uint8 checker x seeded Perlin gradient noise;
* cameras on a horizontal arc around the origin (world +y is down,
  scenegen.py:216-223), looking at the arc axis;
* depth = camera-frame z quantised to uint16 millimetres (core.py:248-257),
  0 = invalid; optional Gaussian noise N(0, (k z)^2) before quantisation;
  invalid pixels either Bernoulli-scattered or drawn from a dilated
  depth-discontinuity band;
* layered inputs exactly as ``conftest.gt_stream_inputs`` builds them
  (tests/conftest.py:28-49): FG pixels Valid, BG pixels Background, injected
  holes and ray misses Invalid; the BG model is the render without FG.

Everything here is test-input infrastructure, run on the host; the same
arrays feed both the GPU path and the CPU oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from .geometry import arc_pose, look_at_pose
from .selection import select_references
from .types import CameraCalibration, CameraIntrinsics, ColorFrame, DepthFrame, Validity

# ---------------------------------------------------------------------------
# procedural texture


class Perlin2:
    """Seeded 2-D gradient noise in [-1, 1]."""

    def __init__(self, seed: int):
        rng = np.random.default_rng(seed)
        self.perm = np.concatenate([rng.permutation(256)] * 2).astype(np.int64)
        ang = rng.uniform(0, 2 * math.pi, 256)
        self.grad = np.stack([np.cos(ang), np.sin(ang)], axis=-1)

    def __call__(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        xi = np.floor(x).astype(np.int64)
        yi = np.floor(y).astype(np.int64)
        xf, yf = x - xi, y - yi
        xi &= 255
        yi &= 255
        p = self.perm

        def g(ix, iy, dx, dy):
            h = p[p[ix] + iy] & 255
            gr = self.grad[h]
            return gr[..., 0] * dx + gr[..., 1] * dy

        def fade(t):
            return t * t * t * (t * (t * 6 - 15) + 10)

        u, v = fade(xf), fade(yf)
        n00 = g(xi, yi, xf, yf)
        n10 = g(xi + 1, yi, xf - 1, yf)
        n01 = g(xi, yi + 1, xf, yf - 1)
        n11 = g(xi + 1, yi + 1, xf - 1, yf - 1)
        a = n00 + u * (n10 - n00)
        b = n01 + u * (n11 - n01)
        return np.clip((a + v * (b - a)) * 1.4, -1.0, 1.0)


@dataclass(frozen=True)
class Texture:
    color_a: tuple
    color_b: tuple
    period: float      # checker period, metres
    noise_scale: float  # Perlin frequency, 1/metres
    seed: int

    def shade(self, s: np.ndarray, t: np.ndarray) -> np.ndarray:
        chk = (np.floor(s / self.period) + np.floor(t / self.period)).astype(np.int64) & 1
        base = np.where(chk[..., None] == 1, np.asarray(self.color_a, float),
                        np.asarray(self.color_b, float))
        n = Perlin2(self.seed)(s * self.noise_scale, t * self.noise_scale)
        return base * (0.8 + 0.2 * n[..., None]) + 18.0 * n[..., None]


# ---------------------------------------------------------------------------
# scene primitives


@dataclass(frozen=True)
class Quad:
    center: np.ndarray
    u_axis: np.ndarray
    v_axis: np.ndarray
    half_u: float
    half_v: float
    tex: Texture


@dataclass(frozen=True)
class Sphere:
    center: np.ndarray
    radius: float
    tex: Texture
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    amp: np.ndarray = field(default_factory=lambda: np.zeros(3))
    freq: float = 0.0
    phase: float = 0.0

    def center_at(self, t: float) -> np.ndarray:
        return self.center + self.velocity * t + self.amp * math.sin(2 * math.pi * self.freq * t
                                                                     + self.phase)


@dataclass(frozen=True)
class Scene:
    quads: tuple
    spheres: tuple
    ground_y: Optional[float]
    ground_tex: Optional[Texture]


def _ray_dirs(calib) -> tuple:
    """World-space ray directions scaled so camera z = 1 (t == depth)."""
    k = calib.intrinsics
    xs = (np.arange(k.width, dtype=np.float64) - k.cx) / k.fx
    ys = (np.arange(k.height, dtype=np.float64) - k.cy) / k.fy
    R = calib.pose.rotation
    # world dir = p_cam @ R with p_cam = (x, y, 1)
    dx = xs[None, :] * R[0, 0] + ys[:, None] * R[1, 0] + R[2, 0]
    dy = xs[None, :] * R[0, 1] + ys[:, None] * R[1, 1] + R[2, 1]
    dz = xs[None, :] * R[0, 2] + ys[:, None] * R[1, 2] + R[2, 2]
    return dx, dy, dz


def render(scene: Scene, calib, t: float = 0.0):
    """Ray cast one camera. Returns dict with float64 depth of the full scene
    (0 = miss), of the background only, the RGB image (uint8) and the FG mask."""
    o = calib.pose.center
    dx, dy, dz = _ray_dirs(calib)
    shape = dx.shape
    inf = np.full(shape, np.inf)
    bg_t, bg_id = inf.copy(), np.full(shape, -1, np.int32)
    # ground plane y = ground_y (world +y down)
    if scene.ground_y is not None:
        with np.errstate(divide="ignore", invalid="ignore"):
            tg = (scene.ground_y - o[1]) / dy
        ok = (dy > 1e-9) & (tg > 1e-6)
        bg_t = np.where(ok, tg, bg_t)
        bg_id = np.where(ok, 0, bg_id)
    for qi, q in enumerate(scene.quads):
        n = np.cross(q.u_axis, q.v_axis)
        den = dx * n[0] + dy * n[1] + dz * n[2]
        with np.errstate(divide="ignore", invalid="ignore"):
            tq = float(np.dot(q.center - o, n)) / den
        px = o[0] + tq * dx - q.center[0]
        py = o[1] + tq * dy - q.center[1]
        pz = o[2] + tq * dz - q.center[2]
        su = px * q.u_axis[0] + py * q.u_axis[1] + pz * q.u_axis[2]
        sv = px * q.v_axis[0] + py * q.v_axis[1] + pz * q.v_axis[2]
        ok = (np.abs(den) > 1e-12) & (tq > 1e-6) & (np.abs(su) <= q.half_u) & \
             (np.abs(sv) <= q.half_v) & (tq < bg_t)
        bg_t = np.where(ok, tq, bg_t)
        bg_id = np.where(ok, 1 + qi, bg_id)
    fg_t, fg_id = inf.copy(), np.full(shape, -1, np.int32)
    centers = []
    for si, s in enumerate(scene.spheres):
        c = s.center_at(t)
        centers.append(c)
        oc = o - c
        a = dx * dx + dy * dy + dz * dz
        b = 2.0 * (dx * oc[0] + dy * oc[1] + dz * oc[2])
        cc = float(np.dot(oc, oc)) - s.radius ** 2
        disc = b * b - 4 * a * cc
        hit = disc > 0
        sq = np.sqrt(np.where(hit, disc, 0.0))
        t0 = (-b - sq) / (2 * a)
        t1 = (-b + sq) / (2 * a)
        ts = np.where(t0 > 1e-6, t0, t1)
        ok = hit & (ts > 1e-6) & (ts < fg_t)
        fg_t = np.where(ok, ts, fg_t)
        fg_id = np.where(ok, si, fg_id)
    fg = fg_t < bg_t
    full_t = np.where(fg, fg_t, bg_t)
    hit_any = np.isfinite(full_t)

    rgb = np.zeros(shape + (3,))
    # background shading evaluated where the BG surface is what the full
    # render sees, and separately nothing is needed for the BG-only model
    for pid in range(-1, len(scene.quads) + 1):
        m = (bg_id == pid) & ~fg & hit_any
        if pid < 0 or not m.any():
            continue
        tt = bg_t[m]
        X = np.stack([o[0] + tt * dx[m], o[1] + tt * dy[m], o[2] + tt * dz[m]], axis=-1)
        if pid == 0:
            rgb[m] = scene.ground_tex.shade(X[:, 0], X[:, 2])
        else:
            q = scene.quads[pid - 1]
            L = X - q.center
            rgb[m] = q.tex.shade(L @ q.u_axis, L @ q.v_axis)
    for si, s in enumerate(scene.spheres):
        m = fg & (fg_id == si)
        if not m.any():
            continue
        tt = fg_t[m]
        L = np.stack([o[0] + tt * dx[m], o[1] + tt * dy[m], o[2] + tt * dz[m]], axis=-1) \
            - centers[si]
        lon = np.arctan2(L[:, 0], L[:, 2]) * s.radius
        lat = np.arcsin(np.clip(L[:, 1] / s.radius, -1, 1)) * s.radius
        rgb[m] = s.tex.shade(lon, lat)
    rgb = np.clip(np.round(rgb), 0, 255).astype(np.uint8)
    return dict(depth=np.where(hit_any, full_t, 0.0), bg_depth=np.where(np.isfinite(bg_t), bg_t, 0.0),
                rgb=rgb, fg=fg & hit_any, hit=hit_any)


# ---------------------------------------------------------------------------
# scene sampling


def _texture(rng, scale: float) -> Texture:
    ca = tuple(int(x) for x in rng.integers(40, 230, 3))
    cb = tuple(int(x) for x in np.clip(np.asarray(ca) + rng.integers(-90, 90, 3), 10, 245))
    return Texture(ca, cb, float(rng.uniform(0.08, 0.3) * scale),
                   float(rng.uniform(2.0, 6.0) / scale), int(rng.integers(1 << 30)))


def _random_in_view(rng, anchor: np.ndarray, d_lo: float, d_hi: float, hspan: float,
                    vspan: float) -> np.ndarray:
    """Point at distance U[d_lo, d_hi] from ``anchor`` inside a view cone along +z."""
    az = math.radians(rng.uniform(-hspan, hspan))
    el = math.radians(rng.uniform(-vspan, vspan))
    d = rng.uniform(d_lo, d_hi)
    direction = np.array([math.sin(az) * math.cos(el), math.sin(el), math.cos(az) * math.cos(el)])
    return anchor + d * direction


def _rig_clearance(c: np.ndarray, arc_radius: float) -> float:
    """Distance from ``c`` to the circle the rig's cameras sit on (radius
    ``arc_radius`` around the world y axis, at y = 0)."""
    return math.hypot(math.hypot(c[0], c[2]) - arc_radius, c[1])


def make_scene(seed: int, n_planes: int, n_spheres: int, plane_dist, sphere_dist,
               sphere_radius, arc_radius: float, ground_y: Optional[float] = None,
               plane_half=(0.4, 1.4), hspan: float = 22.0, vspan: float = 10.0,
               motion: bool = False, near: bool = False) -> Scene:
    """Seeded planes (static BG) and spheres (FG) at the given distances from
    the rig's central camera.

    ``near=True`` is the placement for object ranges that start close to the
    rig (BASELINE.json c1-c4: "0.5-6 m", "0.5-8 m"): a plane's half-sizes are
    ``plane_half`` x its distance (a constant angular size, so a plane 0.5 m
    from the camera is a small card rather than a wall over the whole view),
    a sphere's radius is at most 0.35 x its distance, and an object is
    re-drawn (up to 64 times) while it would reach within 0.45 m of the
    camera arc (where rig and jittered virtual cameras sit)."""
    rng = np.random.default_rng(seed)
    anchor = np.array([0.0, 0.0, -arc_radius])
    quads = []
    for _ in range(n_planes):
        for _try in range(64):
            c = _random_in_view(rng, anchor, *plane_dist, hspan, vspan)
            n = rng.normal(size=3)
            n /= np.linalg.norm(n)
            if n[2] > 0:          # face the rig (normal toward -z)
                n = -n
            if n[2] > -0.6:       # avoid grazing planes
                n[2] = -0.6
                n /= np.linalg.norm(n)
            u = np.cross(n, rng.normal(size=3))
            u /= np.linalg.norm(u)
            v = np.cross(n, u)
            hu, hv = float(rng.uniform(*plane_half)), float(rng.uniform(*plane_half))
            if not near:
                break
            d = float(np.linalg.norm(c - anchor))
            hu, hv = hu * d, hv * d
            if _rig_clearance(c, arc_radius) >= math.hypot(hu, hv) + 0.45:
                break
        quads.append(Quad(c, u, v, hu, hv, _texture(rng, 1.0)))
    spheres = []
    for _ in range(n_spheres):
        for _try in range(64):
            c = _random_in_view(rng, anchor, *sphere_dist, hspan * 0.8, vspan * 0.8)
            rad = float(rng.uniform(*sphere_radius))
            if near:
                rad = min(rad, 0.35 * float(np.linalg.norm(c - anchor)))
            if ground_y is not None:
                c[1] = min(c[1], ground_y - rad - 0.02)
            if not near or _rig_clearance(c, arc_radius) >= rad + 0.45:
                break
        vel = amp = np.zeros(3)
        freq = phase = 0.0
        if motion:
            vel = rng.normal(size=3) * np.array([1.0, 0.1, 1.0])
            vel *= rng.uniform(0.1, 0.6) / max(np.linalg.norm(vel), 1e-9)
            amp = rng.uniform(-0.15, 0.15, 3) * np.array([1.0, 0.3, 1.0])
            freq = float(rng.uniform(0.1, 0.4))
            phase = float(rng.uniform(0, 2 * math.pi))
            # |v| + 2 pi f |a| stays below 1 m/s
            if near:
                # a stream's 10 s (300 frames at 30 fps) keep clear of the arc
                probe = Sphere(c, rad, None, vel, amp, freq, phase)
                for _try in range(8):
                    if all(_rig_clearance(probe.center_at(t), arc_radius) >= rad + 0.45
                           for t in np.linspace(0.0, 10.0, 41)):
                        break
                    vel = vel * 0.5
                    amp = amp * 0.5
                    probe = Sphere(c, rad, None, vel, amp, freq, phase)
        spheres.append(Sphere(c, rad, _texture(rng, 0.5), vel, amp, freq, phase))
    gtex = _texture(rng, 1.5) if ground_y is not None else None
    return Scene(tuple(quads), tuple(spheres), ground_y, gtex)


# ---------------------------------------------------------------------------
# capture: mm quantisation, noise, invalid pixels


def to_mm(depth: np.ndarray) -> np.ndarray:
    """core.depth_to_millimeters semantics: rint, clip [1, 65535], 0 = no depth."""
    mm = np.zeros(depth.shape, dtype=np.uint16)
    ok = depth > 0
    mm[ok] = np.clip(np.round(depth[ok] * 1000.0), 1, 65535).astype(np.uint16)
    return mm


def mm_to_depth(mm: np.ndarray) -> np.ndarray:
    """Metric float32 depth of a mm raster (core.py:264), for building DepthFrames."""
    return mm.astype(np.float32) / np.float32(1000.0)


def _dilate(mask: np.ndarray, r: int) -> np.ndarray:
    out = mask.copy()
    h, w = mask.shape
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            if dy or dx:
                out[max(dy, 0):h + min(dy, 0), max(dx, 0):w + min(dx, 0)] |= \
                    mask[max(-dy, 0):h - max(dy, 0), max(-dx, 0):w - max(dx, 0)]
    return out


@dataclass
class CameraCapture:
    """What one camera delivers to the edge server for one frame."""

    calib: CameraCalibration
    rgb: np.ndarray            # (H, W, 3) uint8
    mm: np.ndarray             # (H, W) uint16, 0 = no depth
    validity: np.ndarray       # (H, W) uint8 sidecar: FG Valid, BG Background, holes Invalid
    bg_depth: np.ndarray       # (H, W) float32 static BG model (from mm)
    bg_validity: np.ndarray    # (H, W) uint8

    def depth_frame(self) -> DepthFrame:
        """The live DepthFrame the reference's mm decode yields (core.py:260-269)."""
        d = mm_to_depth(self.mm)
        v = self.validity.copy()
        v[(v == Validity.VALID) & (self.mm == 0)] = Validity.INVALID
        d[v != Validity.VALID] = 0.0
        H, W = self.mm.shape
        return DepthFrame(W, H, d, v)

    def bg_frame(self) -> DepthFrame:
        H, W = self.mm.shape
        return DepthFrame(W, H, self.bg_depth, self.bg_validity)

    def color_frame(self) -> ColorFrame:
        H, W = self.mm.shape
        return ColorFrame(W, H, self.rgb)


def capture(scene: Scene, calib, seed: int, t: float = 0.0, noise_rel: float = 0.0,
            invalid_frac: float = 0.0, invalid_mode: str = "random",
            layered: bool = True) -> CameraCapture:
    rng = np.random.default_rng(seed)
    r = render(scene, calib, t)
    z = r["depth"]
    if noise_rel > 0:
        z = np.where(r["hit"], z + rng.normal(size=z.shape) * noise_rel * z, 0.0)
        z = np.where(z > 0, z, 0.0)
    mm = to_mm(z)
    if layered:
        validity = np.where(r["fg"], Validity.VALID, Validity.BACKGROUND).astype(np.uint8)
    else:
        validity = np.full(z.shape, Validity.VALID, np.uint8)
    validity[~r["hit"]] = Validity.INVALID
    if invalid_frac > 0:
        n = int(round(invalid_frac * z.size))
        if invalid_mode == "edges":
            zz = np.where(r["hit"], z, 0.0)
            gx = np.zeros_like(zz, dtype=bool)
            gy = np.zeros_like(zz, dtype=bool)
            gx[:, 1:] = np.abs(zz[:, 1:] - zz[:, :-1]) > 0.03 * np.maximum(zz[:, 1:], zz[:, :-1])
            gy[1:, :] = np.abs(zz[1:, :] - zz[:-1, :]) > 0.03 * np.maximum(zz[1:, :], zz[:-1, :])
            band = _dilate(gx | gy, 2)
            cand = np.flatnonzero(band)
            pick = cand if cand.size <= n else rng.choice(cand, n, replace=False)
            kill = np.zeros(z.size, bool)
            kill[pick] = True
            kill = kill.reshape(z.shape)
            mm[kill] = 0
            validity[kill] = Validity.INVALID
        else:
            kill = rng.random(z.shape) < invalid_frac
            mm[kill] = 0       # "2% of depth pixels randomly zeroed" -> Invalid after decode
    if layered:
        mm[validity == Validity.BACKGROUND] = 0   # BG depth travels as the static model
    bg_mm = to_mm(r["bg_depth"]) if layered else np.zeros(z.shape, np.uint16)
    bg_valid = np.where(bg_mm > 0, Validity.VALID, Validity.INVALID).astype(np.uint8)
    bg_depth = np.where(bg_mm > 0, mm_to_depth(bg_mm), np.float32(0.0)).astype(np.float32)
    return CameraCapture(calib, r["rgb"], mm, validity, bg_depth, bg_valid)


# ---------------------------------------------------------------------------
# BASELINE.json configs


@dataclass
class Workload:
    name: str
    seed: int
    rig: List[CameraCalibration]
    virtuals: List[CameraCalibration]
    refs: List[List[int]]                 # per virtual view, reference ids in order
    frames: List[Dict[int, CameraCapture]]  # per frame: camera id -> capture
    description: str = ""

    def inputs(self, frame: int = 0, ids: Optional[Sequence[int]] = None) -> dict:
        """``{id: CameraStreamInputs-like}`` with decoded live DepthFrames."""
        from .synthesis import CameraStreamInputs

        caps = self.frames[frame]
        ids = list(caps) if ids is None else ids
        return {i: CameraStreamInputs(caps[i].calib, caps[i].color_frame(),
                                      caps[i].depth_frame(), caps[i].bg_frame()) for i in ids}


def _intr(w, h, f):
    return CameraIntrinsics(float(f), float(f), w / 2.0, h / 2.0, w, h)


def _arc(n, radius, gap_deg, intr, first_id=0):
    gap = math.radians(gap_deg)
    return [CameraCalibration(first_id + i, intr, arc_pose(radius, (i - (n - 1) / 2.0) * gap))
            for i in range(n)]


CONFIGS = ("c0", "c1", "c2", "c3", "c4")


def workload_params(name: str, seed: int = 2007) -> dict:
    """Rig, scene and capture parameters of config ``name`` (c0..c4) at full size."""
    if name == "c0":
        w, h, f, n, radius, gap = 640, 360, 470.0, 2, 2.5, 15.0
        scene = make_scene(seed, 4, 3, (1.5, 4.0), (1.5, 3.0), (0.2, 0.5), radius,
                           ground_y=None, hspan=25, vspan=12)
        cap = dict(noise_rel=0.0, invalid_frac=0.02, invalid_mode="random")
        phis = [0.0]
        nv, nf, k = 1, 1, 2
    elif name in ("c1", "c2", "c3"):
        w, h, f, n, radius, gap = 1920, 1080, 1400.0, 9, 3.0, 10.0
        # BASELINE.json configs[1]: "6 planes + 5 spheres + a ground plane at 0.5-6 m"
        scene = make_scene(seed, 6, 5, (0.5, 6.0), (0.5, 6.0), (0.15, 0.5), radius,
                           ground_y=1.2, plane_half=(0.15, 0.4), hspan=28, vspan=14,
                           motion=(name == "c3"), near=True)
        cap = dict(noise_rel=0.005, invalid_frac=0.03, invalid_mode="edges")
        k = 3
        if name == "c1":
            phis, nv, nf = [math.radians(5.0)], 1, 1
        elif name == "c2":
            nv, nf, phis = 64, 1, None
        else:
            nv, nf, phis = 300, 300, None
    elif name == "c4":
        w, h, f, n, radius, gap = 3840, 2160, 2800.0, 16, 3.0, 8.0
        # BASELINE.json configs[4]: "40 spheres and 10 planes at 0.5-8 m"
        scene = make_scene(seed, 10, 40, (0.5, 8.0), (0.5, 8.0), (0.1, 0.45), radius,
                           ground_y=1.2, plane_half=(0.1, 0.3), hspan=40, vspan=16, near=True)
        cap = dict(noise_rel=0.005, invalid_frac=0.05, invalid_mode="edges")
        nv, nf, k = 32, 1, 4
        phis = None
    else:
        raise ValueError(f"unknown config {name!r}; expected one of {CONFIGS}")
    return dict(w=w, h=h, f=f, n=n, radius=radius, gap=gap, scene=scene, capture=cap, k=k,
                n_views=nv, n_frames=nf, phis=phis)


def make_workload(name: str, seed: int = 2007, scale: int = 1, n_frames: Optional[int] = None,
                  n_views: Optional[int] = None, cameras: str = "refs",
                  render_frames: bool = True,
                  frame_ids: Optional[Sequence[int]] = None) -> Workload:
    """Build config ``name`` (c0..c4). ``scale`` > 1 divides the resolution
    (for CPU-sized parity cases); ``cameras='refs'`` renders only the cameras
    some view references, ``'all'`` the whole rig. ``n_frames`` overrides the
    frame count of c3; ``render_frames=False`` returns rig, views and
    references without ray-casting any frame (scenes_gpu renders them);
    ``frame_ids`` renders only those frames of the stream (``frames[i]`` is
    then frame ``frame_ids[i]``, still at time ``frame_ids[i] / 30`` s)."""
    prm = workload_params(name, seed)
    w, h, f, n = prm["w"], prm["h"], prm["f"], prm["n"]
    radius, gap, scene, cap, k = prm["radius"], prm["gap"], prm["scene"], prm["capture"], prm["k"]
    nv, nf, phis = prm["n_views"], prm["n_frames"], prm["phis"]
    if name in ("c2", "c4") and n_views:
        nv = n_views
    if name == "c3" and n_frames:
        nf = nv = n_frames
    if not render_frames:
        nf = 0
    if scale > 1:
        w, h, f = w // scale // 2 * 2, h // scale // 2 * 2, f / scale
    intr = _intr(w, h, f)
    rig = _arc(n, radius, gap, intr)
    rng = np.random.default_rng(seed + 17)
    virtuals = []
    if name == "c2" or name == "c4":
        span = (n - 1) * gap / 2.0
        for i in range(nv):
            phi = math.radians(rng.uniform(-span, span))
            rr = radius + rng.uniform(-0.2, 0.2)
            hh = rng.uniform(-0.2, 0.2)
            virtuals.append(CameraCalibration(100 + i, intr, arc_pose(rr, phi, hh)))
    elif name == "c3":
        span = (n - 1) * gap / 2.0
        for i in range(nv):
            phi = math.radians(-span + 2 * span * (i / max(nv - 1, 1)))
            virtuals.append(CameraCalibration(100 + i, intr, arc_pose(radius, phi)))
    else:
        virtuals = [CameraCalibration(100, intr, arc_pose(radius, p)) for p in phis]
    ids = [c.id for c in rig]
    refs = [select_references(v.pose, rig, ids, k) for v in virtuals]
    need = sorted({i for r in refs for i in r}) if cameras == "refs" else ids
    frames = []
    for fi in (range(nf) if frame_ids is None else frame_ids):
        t = fi / 30.0
        view_ids = set(refs[fi]) if name == "c3" and cameras == "refs" else set(need)
        frames.append({cid: capture(scene, rig[cid], seed * 1_000_003 + cid * 7919 + fi, t,
                                    **cap) for cid in sorted(view_ids)})
    desc = f"{name}: {w}x{h}, {n} cams, {k} refs/view, {nv} views, {nf} frames, seed {seed}"
    return Workload(name, seed, rig, virtuals, refs, frames, desc)

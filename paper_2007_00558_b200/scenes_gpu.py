"""Device-side ray caster for the large synthetic workloads.

``scenes.render`` / ``scenes.capture`` ray-cast BASELINE.json's scenes with
numpy on the host, which takes minutes per frame set at 1080p x 300 frames
(c3) or 4K x 16 cameras x 50 primitives (c4). This module evaluates the same
scene description with the same float64 formulas as torch tensor operations
on the GPU, so those workloads are generated in HBM in seconds and never cross
PCIe. It is test-input infrastructure like ``scenes``: nothing on the
synthesis path imports it.

Equivalence with the host generator: the ray/primitive intersection, texture
and mm quantisation formulas are the same (tests/test_host.py compares both at
reduced size: depth rasters equal, RGB equal up to the rounding of libm vs
torch transcendental ulps). Noise and invalid-pixel draws come from a torch
generator seeded like ``capture``'s numpy one, so they are seeded and
reproducible but not the same samples.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np
import torch

from . import scenes
from .types import Validity


class _Perlin:
    """scenes.Perlin2 with its permutation/gradient tables on the device."""

    def __init__(self, seed: int, dev):
        p = scenes.Perlin2(seed)
        self.perm = torch.from_numpy(p.perm).to(dev)
        self.grad = torch.from_numpy(p.grad).to(dev)

    def __call__(self, x, y):
        xi = torch.floor(x)
        yi = torch.floor(y)
        xf, yf = x - xi, y - yi
        xi = xi.to(torch.int64) & 255
        yi = yi.to(torch.int64) & 255
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
        return torch.clamp((a + v * (b - a)) * 1.4, -1.0, 1.0)


def _shade(tex, s, t, dev, cache):
    """scenes.Texture.shade on the device."""
    chk = (torch.floor(s / tex.period) + torch.floor(t / tex.period)).to(torch.int64) & 1
    ca = torch.tensor(tex.color_a, dtype=torch.float64, device=dev)
    cb = torch.tensor(tex.color_b, dtype=torch.float64, device=dev)
    base = torch.where(chk[..., None] == 1, ca, cb)
    pn = cache.get(tex.seed)
    if pn is None:
        pn = cache[tex.seed] = _Perlin(tex.seed, dev)
    n = pn(s * tex.noise_scale, t * tex.noise_scale)
    return base * (0.8 + 0.2 * n[..., None]) + 18.0 * n[..., None]


def _ray_dirs(calib, dev):
    k = calib.intrinsics
    xs = (torch.arange(k.width, dtype=torch.float64, device=dev) - k.cx) / k.fx
    ys = (torch.arange(k.height, dtype=torch.float64, device=dev) - k.cy) / k.fy
    R = [float(x) for x in np.asarray(calib.pose.rotation, np.float64).ravel()]
    dx = xs[None, :] * R[0] + ys[:, None] * R[3] + R[6]
    dy = xs[None, :] * R[1] + ys[:, None] * R[4] + R[7]
    dz = xs[None, :] * R[2] + ys[:, None] * R[5] + R[8]
    return dx, dy, dz


def render(scene, calib, t: float = 0.0, dev="cuda", cache=None):
    """scenes.render on the device: dict of depth (f64, 0 = miss), bg_depth,
    rgb (u8), fg and hit masks, all torch tensors on ``dev``."""
    cache = {} if cache is None else cache
    o = [float(x) for x in np.asarray(calib.pose.center, np.float64)]
    dx, dy, dz = _ray_dirs(calib, dev)
    shape = dx.shape
    inf = torch.full(shape, math.inf, dtype=torch.float64, device=dev)
    bg_t = inf.clone()
    bg_id = torch.full(shape, -1, dtype=torch.int32, device=dev)
    if scene.ground_y is not None:
        tg = (scene.ground_y - o[1]) / dy
        ok = (dy > 1e-9) & (tg > 1e-6)
        bg_t = torch.where(ok, tg, bg_t)
        bg_id = torch.where(ok, torch.zeros_like(bg_id), bg_id)
    for qi, q in enumerate(scene.quads):
        n = np.cross(q.u_axis, q.v_axis)
        den = dx * n[0] + dy * n[1] + dz * n[2]
        tq = float(np.dot(q.center - np.asarray(o), n)) / den
        px = o[0] + tq * dx - q.center[0]
        py = o[1] + tq * dy - q.center[1]
        pz = o[2] + tq * dz - q.center[2]
        su = px * q.u_axis[0] + py * q.u_axis[1] + pz * q.u_axis[2]
        sv = px * q.v_axis[0] + py * q.v_axis[1] + pz * q.v_axis[2]
        ok = (den.abs() > 1e-12) & (tq > 1e-6) & (su.abs() <= q.half_u) & \
             (sv.abs() <= q.half_v) & (tq < bg_t)
        bg_t = torch.where(ok, tq, bg_t)
        bg_id = torch.where(ok, torch.full_like(bg_id, 1 + qi), bg_id)
    fg_t = inf.clone()
    fg_id = torch.full(shape, -1, dtype=torch.int32, device=dev)
    centers = []
    a = dx * dx + dy * dy + dz * dz
    for si, s in enumerate(scene.spheres):
        c = s.center_at(t)
        centers.append(c)
        oc = np.asarray(o) - c
        b = 2.0 * (dx * oc[0] + dy * oc[1] + dz * oc[2])
        cc = float(np.dot(oc, oc)) - s.radius ** 2
        disc = b * b - 4 * a * cc
        hit = disc > 0
        sq = torch.sqrt(torch.where(hit, disc, torch.zeros_like(disc)))
        t0 = (-b - sq) / (2 * a)
        t1 = (-b + sq) / (2 * a)
        ts = torch.where(t0 > 1e-6, t0, t1)
        ok = hit & (ts > 1e-6) & (ts < fg_t)
        fg_t = torch.where(ok, ts, fg_t)
        fg_id = torch.where(ok, torch.full_like(fg_id, si), fg_id)
    fg = fg_t < bg_t
    full_t = torch.where(fg, fg_t, bg_t)
    hit_any = torch.isfinite(full_t)

    rgb = torch.zeros(shape + (3,), dtype=torch.float64, device=dev)
    for pid in range(0, len(scene.quads) + 1):
        m = (bg_id == pid) & ~fg & hit_any
        if not bool(m.any()):
            continue
        tt = bg_t[m]
        X = torch.stack([o[0] + tt * dx[m], o[1] + tt * dy[m], o[2] + tt * dz[m]], dim=-1)
        if pid == 0:
            rgb[m] = _shade(scene.ground_tex, X[:, 0], X[:, 2], dev, cache)
        else:
            q = scene.quads[pid - 1]
            L = X - torch.from_numpy(np.asarray(q.center, np.float64)).to(dev)
            ua = torch.from_numpy(np.asarray(q.u_axis, np.float64)).to(dev)
            va = torch.from_numpy(np.asarray(q.v_axis, np.float64)).to(dev)
            rgb[m] = _shade(q.tex, L @ ua, L @ va, dev, cache)
    for si, s in enumerate(scene.spheres):
        m = fg & (fg_id == si)
        if not bool(m.any()):
            continue
        tt = fg_t[m]
        L = torch.stack([o[0] + tt * dx[m], o[1] + tt * dy[m], o[2] + tt * dz[m]], dim=-1) \
            - torch.from_numpy(np.asarray(centers[si], np.float64)).to(dev)
        lon = torch.atan2(L[:, 0], L[:, 2]) * s.radius
        lat = torch.asin(torch.clamp(L[:, 1] / s.radius, -1, 1)) * s.radius
        rgb[m] = _shade(s.tex, lon, lat, dev, cache)
    rgb = torch.clamp(torch.round(rgb), 0, 255).to(torch.uint8)
    zero = torch.zeros_like(full_t)
    return dict(depth=torch.where(hit_any, full_t, zero),
                bg_depth=torch.where(torch.isfinite(bg_t), bg_t, zero),
                rgb=rgb, fg=fg & hit_any, hit=hit_any)


def to_mm(depth):
    """scenes.to_mm on the device (rint half-even, clip [1, 65535], 0 = none);
    returned as int16 holding the uint16 bit pattern (torch has no uint16 math)."""
    mm = torch.clamp(torch.round(depth * 1000.0), 1, 65535)
    mm = torch.where(depth > 0, mm, torch.zeros_like(mm)).to(torch.int32)
    return (mm - ((mm >> 15) << 16)).to(torch.int16)


def mm_to_depth(mm16):
    return (mm16.to(torch.int32) & 0xFFFF).to(torch.float32) / torch.tensor(1000.0,
                                                                            dtype=torch.float32)


@dataclass
class DeviceCapture:
    """scenes.CameraCapture with device tensors (mm as int16 bit pattern)."""

    calib: object
    rgb: torch.Tensor
    mm: torch.Tensor
    validity: torch.Tensor
    bg_depth: torch.Tensor
    bg_validity: torch.Tensor

    def host(self) -> scenes.CameraCapture:
        return scenes.CameraCapture(self.calib, self.rgb.cpu().numpy(),
                                    self.mm.cpu().numpy().view(np.uint16),
                                    self.validity.cpu().numpy(), self.bg_depth.cpu().numpy(),
                                    self.bg_validity.cpu().numpy())


def _dilate(mask, r: int):
    m = mask[None, None].to(torch.float32)
    return torch.nn.functional.max_pool2d(m, 2 * r + 1, stride=1, padding=r)[0, 0] > 0


def capture(scene, calib, seed: int, t: float = 0.0, noise_rel: float = 0.0,
            invalid_frac: float = 0.0, invalid_mode: str = "random", layered: bool = True,
            dev="cuda", cache=None) -> DeviceCapture:
    """scenes.capture on the device (noise / invalid draws from a seeded torch
    generator)."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) & ((1 << 63) - 1))
    r = render(scene, calib, t, dev, cache)
    z = r["depth"]
    hit = r["hit"]
    if noise_rel > 0:
        nz = torch.randn(z.shape, generator=gen, dtype=torch.float64, device=dev)
        z = torch.where(hit, z + nz * noise_rel * z, torch.zeros_like(z))
        z = torch.where(z > 0, z, torch.zeros_like(z))
    mm = to_mm(z)
    if layered:
        validity = torch.where(r["fg"], Validity.VALID, Validity.BACKGROUND).to(torch.uint8)
    else:
        validity = torch.full(z.shape, Validity.VALID, dtype=torch.uint8, device=dev)
    validity[~hit] = Validity.INVALID
    if invalid_frac > 0:
        n = int(round(invalid_frac * z.numel()))
        if invalid_mode == "edges":
            zz = torch.where(hit, z, torch.zeros_like(z))
            gx = torch.zeros_like(zz, dtype=torch.bool)
            gy = torch.zeros_like(zz, dtype=torch.bool)
            gx[:, 1:] = (zz[:, 1:] - zz[:, :-1]).abs() > 0.03 * torch.maximum(zz[:, 1:], zz[:, :-1])
            gy[1:, :] = (zz[1:, :] - zz[:-1, :]).abs() > 0.03 * torch.maximum(zz[1:, :], zz[:-1, :])
            cand = torch.nonzero(_dilate(gx | gy, 2).flatten()).flatten()
            if cand.numel() > n:
                cand = cand[torch.randperm(cand.numel(), generator=gen, device=dev)[:n]]
            kill = torch.zeros(z.numel(), dtype=torch.bool, device=dev)
            kill[cand] = True
            kill = kill.view(z.shape)
            mm[kill] = 0
            validity[kill] = Validity.INVALID
        else:
            kill = torch.rand(z.shape, generator=gen, device=dev) < invalid_frac
            mm[kill] = 0
    if layered:
        mm[validity == Validity.BACKGROUND] = 0
        bg_mm = to_mm(r["bg_depth"])
    else:
        bg_mm = torch.zeros_like(mm)
    bg_ok = bg_mm != 0
    bg_valid = torch.where(bg_ok, Validity.VALID, Validity.INVALID).to(torch.uint8)
    bg_depth = torch.where(bg_ok, mm_to_depth(bg_mm), torch.zeros((), dtype=torch.float32,
                                                                   device=dev))
    return DeviceCapture(calib, r["rgb"], mm, validity, bg_depth, bg_valid)


def make_workload(name: str, seed: int = 2007, n_frames: Optional[int] = None,
                  n_views: Optional[int] = None, cameras: str = "refs", dev="cuda",
                  scale: int = 1, frame_ids=None) -> scenes.Workload:
    """scenes.make_workload with the frames rendered on ``dev`` (DeviceCapture
    values). Rig, virtual cameras, reference lists and the scene are the host
    generator's own (same seed -> same geometry). ``frame_ids`` (c3) renders
    only those frames of the stream: ``frames[i]`` is frame ``frame_ids[i]``
    (a rank renders only the frames it owns)."""
    skel = scenes.make_workload(name, seed=seed, scale=scale, n_frames=n_frames,
                                n_views=n_views, cameras=cameras, render_frames=False)
    params = scenes.workload_params(name, seed)
    cache: Dict[int, _Perlin] = {}
    nf = len(skel.virtuals) if name == "c3" else 1
    frames: List[Dict[int, DeviceCapture]] = []
    ids = [c.id for c in skel.rig]
    need = sorted({i for r in skel.refs for i in r}) if cameras == "refs" else ids
    for fi in (range(nf) if frame_ids is None else frame_ids):
        view_ids = set(skel.refs[fi]) if name == "c3" and cameras == "refs" else set(need)
        frames.append({cid: capture(params["scene"], skel.rig[cid],
                                    seed * 1_000_003 + cid * 7919 + fi, fi / 30.0,
                                    dev=dev, cache=cache, **params["capture"])
                       for cid in sorted(view_ids)})
    desc = skel.description.replace(" 0 frames", f" {nf} frames") + " (frames ray-cast on the GPU)"
    if frame_ids is not None:
        desc += f", {len(frames)} of them rendered here"
    return scenes.Workload(skel.name, seed, skel.rig, skel.virtuals, skel.refs, frames, desc)

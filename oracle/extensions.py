"""CPU restatement of the library's two EXTENSIONS (test infrastructure only).

Neither exists in the reference (blend weights are
baseline-only, synthesis.py:249,257; holes keep hole_color, synthesis.py:
308-311). The north star asks for both, so the library offers
them off by default (``SynthesisConfig.angular_weight`` / ``inpaint``); this
module states what they compute so the GPU tests have a checker:

* ``angular_mix`` — mix_layer (synthesis.py:261-292) with the per-pixel weight
  w_j * 1 / (theta_j + eps), theta_j the angle at the surface point between
  the rays to reference camera j and to the virtual camera;
* ``inpaint`` — K4's background-biased fill of composite holes.

There is no reference implementation to pin these against; they restate the
kernels' own definitions (paper_2007_00558_b200/csrc/fvv_kernels.cu,
``angular_factor`` and ``k_inpaint``).
"""

from __future__ import annotations

import numpy as np

from .fvv_oracle import Cam, rays


def angular_factor(virtual, src, z, eps):
    """1 / (theta + eps) per pixel of the virtual view at depth z (H, W)."""
    v, s = Cam(virtual), Cam(src)
    rx, ry = rays(v)
    px, py, pz = rx[None, :] * z, ry[:, None] * z, z
    wx = px * v.R[0, 0] + py * v.R[1, 0] + pz * v.R[2, 0] + v.C[0]
    wy = px * v.R[0, 1] + py * v.R[1, 1] + pz * v.R[2, 1] + v.C[1]
    wz = px * v.R[0, 2] + py * v.R[1, 2] + pz * v.R[2, 2] + v.C[2]
    a = np.stack([wx - s.C[0], wy - s.C[1], wz - s.C[2]], -1)
    b = np.stack([wx - v.C[0], wy - v.C[1], wz - v.C[2]], -1)
    den = np.sqrt(np.sum(a * a, -1) * np.sum(b * b, -1))
    with np.errstate(invalid="ignore", divide="ignore"):
        cs = np.where(den > 0, np.sum(a * b, -1) / den, 1.0)
    # the kernel evaluates the arccos in single precision
    theta = np.arccos(np.clip(cs, -1.0, 1.0).astype(np.float32)).astype(np.float64)
    return 1.0 / (theta + eps)


def angular_mix(contribs, virtual, srcs, weights, band_rel, eps):
    """mix_layer with per-pixel angular weights; contribs = [(color, depth, valid)]."""
    H, W = contribs[0][1].shape
    zmin = np.full((H, W), np.inf)
    for _, d, v in contribs:
        zmin = np.where(v & (d < zmin), d, zmin)
    thr = zmin + band_rel * zmin
    acc = np.zeros((H, W, 3))
    wacc = np.zeros((H, W))
    for (c, d, v), s, w in zip(contribs, srcs, weights):
        part = v & (d <= thr)
        wp = w * angular_factor(virtual, s, np.where(v, d, 1.0), eps)
        acc += np.where(part[..., None], wp[..., None] * c, 0.0)
        wacc += np.where(part, wp, 0.0)
    valid = wacc > 0
    with np.errstate(invalid="ignore", divide="ignore"):
        col = np.where(valid[..., None], acc / np.where(valid, wacc, 1.0)[..., None], 0.0)
    return col, valid


def inpaint(rgb, prov, depth, radius=64, bg_band=0.05):
    """K4: each hole (prov 0) takes the first non-hole pixel (prov 1 or 2) to
    its left, right, top and bottom within `radius`, keeps those whose depth
    is within bg_band of the farthest one and averages their colours with
    1/distance weights (f32, in that order). Returns (rgb, prov)."""
    rgb = rgb.copy()
    out_prov = prov.copy()
    H, W = prov.shape
    src_rgb = rgb.copy()
    dirs = [(-1, 0), (1, 0), (0, -1), (0, 1)]   # left, right, up, down
    for y, x in zip(*np.nonzero(prov == 0)):
        cands = []
        for dx, dy in dirs:
            xx, yy = x, y
            for s in range(1, radius + 1):
                xx += dx
                yy += dy
                if not (0 <= xx < W and 0 <= yy < H):
                    break
                if prov[yy, xx] in (1, 2):
                    cands.append((np.float32(depth[yy, xx]), np.float32(s), src_rgb[yy, xx]))
                    break
        if not cands:
            continue
        zmax = max(c[0] for c in cands)
        zlo = np.float32(zmax * np.float32(1.0 - bg_band))
        acc = np.zeros(3, np.float32)
        aw = np.float32(0)
        for z, dist, c in cands:
            if z < zlo:
                continue
            w = np.float32(1.0) / dist
            acc += w * c.astype(np.float32)
            aw += w
        rgb[y, x] = np.clip(np.rint(acc / aw), 0, 255).astype(np.uint8)
        out_prov[y, x] = 3
    return rgb, out_prov

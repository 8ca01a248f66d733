"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's edge-server view-synthesis path
(``/root/reference/pkg/src/fvv``), used as the checker for the sm_100a
kernels. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it; the product
package never does (it fails loudly when its CUDA library is missing).

What it restates, function by function (each cites the reference line):

* ``decode_mm``            core.depth_from_millimeters      core.py:260-269
* ``unpack_yuv420``        depthcodec.unpack_yuv420         depthcodec.py:154-177,213-222
* ``dequantize12``         depthcodec.dequantize12/_codes   depthcodec.py:113-138
* ``bilateral_close_holes`` depthproc.bilateral_close_holes depthproc.py:171-224
* ``forward_warp``         synthesis.warp_layer stage 1     synthesis.py:184-205
* ``resolve_zbuf``         warp_layer splat policy + crack  synthesis.py:79-125,207-222
* ``backward_fetch``       warp_layer stage 3 + bilinear    synthesis.py:128-159,224-247
* ``warp_layer``           synthesis.warp_layer             synthesis.py:162-258
* ``mix_layer``            synthesis.mix_layer              synthesis.py:261-292
* ``composite``            synthesis.composite              synthesis.py:295-318
* ``synthesize_view``      synthesis.synthesize_view        synthesis.py:331-362
* ``quantize12`` / ``pack_yuv420``  depthcodec encoder       depthcodec.py:83-110,141-193
* ``correct_depth``        depthproc.correct_depth          depthproc.py:67-84
* ``bg_train`` / ``classify_fg``  depthproc BG model         depthproc.py:121-149
* ``remove_bg_depth``      depthproc.remove_bg_depth        depthproc.py:152-164
* ``depth_to_millimeters`` core.depth_to_millimeters        core.py:246-255
* ``rle_encode`` / ``rle_decode``  mvdio validity sidecar   mvdio.py:34-52

Differences from the reference, all deliberate and mirrored by the kernels:

1. Geometry is evaluated element-wise in a fixed order with no FMA
   contraction, e.g. ``X = ((px*R00 + py*R10) + pz*R20) + C0``, instead of the
   reference's BLAS ``@`` (core.py:163,169). The two agree to the last ulp in
   most coordinates and on every rounded target pixel the survey probed
   (SURVEY.md §0, App. B). This makes the oracle reproducible bit for bit on
   any machine, which the BLAS path is not.
2. The z-buffer (``np.minimum.at`` on float64 z, synthesis.py:196-205) is
   restated as ONE scatter per source into a canvas padded by ``r`` followed by
   a (2r+1)^2-1 ring min (verified equivalent), on a 64-bit
   key ``zcode << b | source_index`` (``b`` = bits of the source pixel count,
   ``zcode`` = 5 exponent bits + (52-b) mantissa bits of z). The winner's exact
   float64 z is recovered from its index. Two sources whose z agree in the
   kept bits (relative gap < 2^-(52-b), ~5e-10 at 1080p) resolve to the lower
   index instead of the smaller z. This gives the winner-index maps the
   north star asks for, which the reference never materialises.

Everything else (rint half-even rounding, fp32 true division for mm, f64
exp for the bilateral range weight, nanmedian's even-count average, the
bilinear clip/band/threshold quirks, strict ``<`` for z_min vs ``<=`` for the
band, ordered accumulation) follows the reference exactly.
"""

from __future__ import annotations

import math

import numpy as np

VALID, INVALID, BACKGROUND = 0, 1, 2

# ----------------------------------------------------------------------------
# z-key format (shared with csrc/fvv_kernels.cuh; see module docstring, item 2)

KEY_GEN_BITS = 7            # top bits: canvas generation (0 here; kernels rotate it)
KEY_EXP_BITS = 5            # exponent window: z in [2^-16, 2^16) metres
KEY_EXP_MIN = 1023 - 16     # biased f64 exponent mapped to zcode exponent 0
KEY_EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)

STAGE_NONE, STAGE_CENTER, STAGE_SPLAT, STAGE_CRACK = 0, 1, 2, 3


def index_bits(n_pixels: int) -> int:
    return max(1, int(n_pixels - 1).bit_length())


def z_keys(z: np.ndarray, idx: np.ndarray, b: int) -> np.ndarray:
    """Key of each (z > 0, source index) pair; generation bits are 0."""
    m = 52 - b
    bits = np.ascontiguousarray(z, dtype=np.float64).view(np.uint64)
    e = ((bits >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64)
    mant = (bits & np.uint64((1 << 52) - 1)) >> np.uint64(52 - m)
    zc = (np.clip(e - KEY_EXP_MIN, 0, 31).astype(np.uint64) << np.uint64(m)) | mant
    zc = np.where(e < KEY_EXP_MIN, np.uint64(0), zc)
    zc = np.where(e > KEY_EXP_MIN + 31, np.uint64((1 << (KEY_EXP_BITS + m)) - 1), zc)
    return (zc << np.uint64(b)) | idx.astype(np.uint64)


# ----------------------------------------------------------------------------
# cameras


class Cam:
    """Plain camera record: intrinsics, world->camera R (3x3), centre C."""

    __slots__ = ("id", "width", "height", "fx", "fy", "cx", "cy", "R", "C")

    def __init__(self, calib):
        k = calib.intrinsics
        self.id = int(calib.id)
        self.width, self.height = int(k.width), int(k.height)
        self.fx, self.fy, self.cx, self.cy = float(k.fx), float(k.fy), float(k.cx), float(k.cy)
        self.R = np.asarray(calib.pose.rotation, dtype=np.float64)
        self.C = np.asarray(calib.pose.center, dtype=np.float64)


def _cam(c):
    return c if isinstance(c, Cam) else Cam(c)


def rays(cam: Cam):
    """Per-column / per-row ray slopes, ``core.py:224-227``."""
    rx = (np.arange(cam.width, dtype=np.float64) - cam.cx) / cam.fx
    ry = (np.arange(cam.height, dtype=np.float64) - cam.cy) / cam.fy
    return rx, ry


def cam_to_world(px, py, pz, cam: Cam):
    """``p @ R + C`` (core.py:166-169), fixed summation order."""
    R, C = cam.R, cam.C
    wx = ((px * R[0, 0] + py * R[1, 0]) + pz * R[2, 0]) + C[0]
    wy = ((px * R[0, 1] + py * R[1, 1]) + pz * R[2, 1]) + C[1]
    wz = ((px * R[0, 2] + py * R[1, 2]) + pz * R[2, 2]) + C[2]
    return wx, wy, wz


def world_to_cam(wx, wy, wz, cam: Cam):
    """``(X - C) @ R.T`` (core.py:160-163), fixed summation order."""
    R, C = cam.R, cam.C
    dx, dy, dz = wx - C[0], wy - C[1], wz - C[2]
    x = (dx * R[0, 0] + dy * R[0, 1]) + dz * R[0, 2]
    y = (dx * R[1, 0] + dy * R[1, 1]) + dz * R[1, 2]
    z = (dx * R[2, 0] + dy * R[2, 1]) + dz * R[2, 2]
    return x, y, z


def relative_pose(src: Cam, dst: Cam):
    """The src-camera -> dst-camera rigid motion, composed once per camera
    pair in a fixed order: ``M = R_dst R_src^T``, ``t = R_dst (C_src - C_dst)``
    (``world_to_camera(camera_to_world(p, src), dst)``, core.py:160-169, is
    ``M p + t``). Python floats: IEEE f64, no fused multiply-add."""
    Rs, Rd = src.R, dst.R
    dc = [float(src.C[k]) - float(dst.C[k]) for k in range(3)]
    M = [[(float(Rd[i, 0]) * float(Rs[j, 0]) + float(Rd[i, 1]) * float(Rs[j, 1]))
          + float(Rd[i, 2]) * float(Rs[j, 2]) for j in range(3)] for i in range(3)]
    t = [(float(Rd[i, 0]) * dc[0] + float(Rd[i, 1]) * dc[1]) + float(Rd[i, 2]) * dc[2]
         for i in range(3)]
    return M, t


def transfer(depth_f64, src: Cam, dst: Cam, us=None, vs=None):
    """Lift src pixels at ``depth`` and express them in dst's camera frame:
    ``unproject_map`` (core.py:230-234) followed by ``world_to_camera``
    (core.py:160-169), as ``M (rx d, ry d, d) + t`` evaluated per coordinate
    i as ``((M_i0 rx) + ((M_i1 ry) + M_i2)) d + t_i`` — the ray (rx, ry, 1)
    is rotated first (its row part once per source row), then scaled by the
    depth. Without ``us``/``vs`` the whole raster is used.
    """
    M, t = relative_pose(src, dst)
    rx, ry = rays(src)
    if us is None:
        RX, RY = rx[None, :], ry[:, None]
    else:
        RX, RY = rx[us], ry[vs]
    out = []
    for i in range(3):
        q = M[i][1] * RY + M[i][2]
        a = M[i][0] * RX + q
        out.append(a * depth_f64 + t[i])
    return tuple(out)


def project(x, y, z, cam: Cam):
    """``u = fx*x/z + cx`` evaluated as ``(fx*x)/z + cx`` (core.py:212-213)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        u = (cam.fx * x) / z + cam.cx
        v = (cam.fy * y) / z + cam.cy
    return u, v


# ----------------------------------------------------------------------------
# K0: depth decode


def decode_mm(mm: np.ndarray, validity: np.ndarray):
    """``core.depth_from_millimeters`` (core.py:260-269): fp32 true division."""
    depth = mm.astype(np.float32) / np.float32(1000.0)
    val = np.asarray(validity, dtype=np.uint8).copy()
    val[(val == VALID) & (mm == 0)] = INVALID
    depth[val != VALID] = 0.0
    return depth, val


def encode_mm(depth: np.ndarray, validity: np.ndarray) -> np.ndarray:
    """``core.depth_to_millimeters`` (core.py:248-257), used to build inputs."""
    mm = np.zeros(depth.shape, dtype=np.uint16)
    ok = validity == VALID
    mm[ok] = np.clip(np.round(depth[ok] * 1000.0), 1, 65535).astype(np.uint16)
    return mm


_DEINT_A = np.zeros(256, dtype=np.uint16)
_DEINT_B = np.zeros(256, dtype=np.uint16)
for _c in range(256):
    for _bit in range(4):
        _DEINT_A[_c] |= ((_c >> (2 * _bit + 1)) & 1) << _bit
        _DEINT_B[_c] |= ((_c >> (2 * _bit)) & 1) << _bit


def unpack_yuv420(y, u, v) -> np.ndarray:
    """12-bit codes from the folded/interleaved YUV420 raster (depthcodec.py:213-222)."""
    h, w = y.shape
    msb = np.empty((h, w), dtype=np.uint16)
    msb[0::2, 0::2] = _DEINT_A[u]
    msb[0::2, 1::2] = _DEINT_B[u]
    msb[1::2, 0::2] = _DEINT_A[v]
    msb[1::2, 1::2] = _DEINT_B[v]
    lsb = np.where(msb % 2 == 0, y.astype(np.uint16), 255 - y.astype(np.uint16))
    return (msb << 8) | lsb.astype(np.uint16)


def pack_yuv420(codes: np.ndarray):
    """Inverse of ``unpack_yuv420`` (depthcodec.py:141-193), for building inputs."""
    msb = (codes >> 8).astype(np.uint8)
    lsb = (codes & 0xFF).astype(np.uint8)
    y = np.where(msb % 2 == 0, lsb, 255 - lsb).astype(np.uint8)

    def inter(a, b):
        out = np.zeros(a.shape, dtype=np.uint8)
        for bit in range(4):
            out |= (((a >> bit) & 1) << (2 * bit + 1)).astype(np.uint8)
            out |= (((b >> bit) & 1) << (2 * bit)).astype(np.uint8)
        return out

    return y, inter(msb[0::2, 0::2], msb[0::2, 1::2]), inter(msb[1::2, 0::2], msb[1::2, 1::2])


def dequantize12(codes: np.ndarray, z_near: float, z_far: float):
    """Codes -> (f32 depth, validity) (depthcodec.py:113-138): f64 formula, f32 cast."""
    inv_span = 1.0 / z_near - 1.0 / z_far
    frac = (codes.astype(np.float64) - 2) / 4093
    with np.errstate(divide="ignore"):
        z = 1.0 / (frac * inv_span + 1.0 / z_far)
    z[codes < 2] = 0.0
    val = np.full(codes.shape, VALID, dtype=np.uint8)
    val[codes == 0] = BACKGROUND
    val[codes == 1] = INVALID
    z[val != VALID] = 0.0
    return z.astype(np.float32), val


def quantize12(depth, validity, z_near, z_far) -> np.ndarray:
    """depthcodec.quantize12 (depthcodec.py:83-110), for building inputs."""
    z = depth.astype(np.float64)
    out = np.full(z.shape, 1, dtype=np.uint16)
    out[validity == BACKGROUND] = 0
    band = (validity == VALID) & (z >= z_near * 0.99) & (z <= z_far * 1.01)
    zc = np.clip(z, z_near, z_far)
    frac = (1.0 / zc - 1.0 / z_far) / (1.0 / z_near - 1.0 / z_far)
    code = np.clip(np.floor(4093 * frac + 2 + 0.5), 2, 4095)
    out[band] = code[band].astype(np.uint16)
    return out


# ----------------------------------------------------------------------------
# K1: joint-bilateral hole closing


def shift2d(a: np.ndarray, dy: int, dx: int) -> np.ndarray:
    """Zero-filled integer shift: out[y, x] = a[y - dy, x - dx] (scenegen.py:392-400)."""
    out = np.zeros_like(a)
    h, w = a.shape[:2]
    out[max(dy, 0):min(h + dy, h), max(dx, 0):min(w + dx, w)] = \
        a[max(-dy, 0):min(h - dy, h), max(-dx, 0):min(w - dx, w)]
    return out


def bilateral_close_holes(depth, validity, rgb, radius=2, sigma_spatial=2.0,
                          sigma_range=10.0, min_valid_neighbors=6):
    """depthproc.bilateral_close_holes (depthproc.py:171-224).

    Returns (depth f32, validity u8, filled mask). With no INVALID pixel the
    inputs come back unchanged (the reference returns the same object).
    """
    holes = validity == INVALID
    if not holes.any():
        return depth, validity, np.zeros(depth.shape, dtype=bool)
    valid = (validity == VALID).astype(np.float64)
    z = depth.astype(np.float64)
    g = rgb.astype(np.float64)
    num = np.zeros(z.shape)
    den = np.zeros(z.shape)
    cnt = np.zeros(z.shape, dtype=np.int32)
    inv_2ss = 1.0 / (2.0 * sigma_spatial ** 2)
    inv_2sr = 1.0 / (2.0 * sigma_range ** 2)
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            if dy == 0 and dx == 0:
                continue
            nb_valid = shift2d(valid, dy, dx) > 0
            nb_z = shift2d(z, dy, dx)
            d0 = g[..., 0] - shift2d(g[..., 0], dy, dx)
            d1 = g[..., 1] - shift2d(g[..., 1], dy, dx)
            d2 = g[..., 2] - shift2d(g[..., 2], dy, dx)
            d2sum = (d0 ** 2 + d1 ** 2) + d2 ** 2
            w = math.exp(-(dy * dy + dx * dx) * inv_2ss) * np.exp(-d2sum * inv_2sr)
            w = np.where(nb_valid, w, 0.0)
            num += w * nb_z
            den += w
            cnt += nb_valid.astype(np.int32)
    fill = holes & (cnt >= min_valid_neighbors) & (den > 0)
    out_d = depth.copy()
    out_v = validity.copy()
    with np.errstate(invalid="ignore", divide="ignore"):
        out_d[fill] = (num[fill] / den[fill]).astype(np.float32)
    out_v[fill] = VALID
    return out_d, out_v, fill


# ----------------------------------------------------------------------------
# K2: forward warp into a keyed z canvas


class Warp:
    """Per-contribution forward-warp state: canvas, per-source z and index bits."""

    def __init__(self, canvas, z_src, b, r, shape):
        self.canvas, self.z_src, self.b, self.r, self.shape = canvas, z_src, b, r, shape


def forward_warp(depth, valid_mask, src, dst, r: int) -> Warp:
    """Stage 1 of warp_layer (synthesis.py:188-205) on the keyed canvas."""
    src, dst = _cam(src), _cam(dst)
    d = depth.astype(np.float64)
    x, y, z = transfer(d, src, dst)
    u, v = project(x, y, z, dst)
    ok = valid_mask & (z > 0)
    ui = np.rint(np.where(ok, u, 0.0))
    vi = np.rint(np.where(ok, v, 0.0))
    ok &= (ui >= -r) & (ui < dst.width + r) & (vi >= -r) & (vi < dst.height + r)
    wc = dst.width + 2 * r
    idx = np.flatnonzero(ok)
    cell = (vi.ravel()[idx].astype(np.int64) + r) * wc + (ui.ravel()[idx].astype(np.int64) + r)
    b = index_bits(src.width * src.height)
    canvas = np.full((dst.height + 2 * r) * wc, KEY_EMPTY, dtype=np.uint64)
    np.minimum.at(canvas, cell, z_keys(z.ravel()[idx], idx, b))
    return Warp(canvas.reshape(dst.height + 2 * r, wc), z.ravel(), b, r,
                (dst.height, dst.width))


def _count8(mask):
    """``_neighbor_count`` (synthesis.py:79-87): 8-neighbourhood, zero padded."""
    m = mask.astype(np.int32)
    return sum(shift2d(m, dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1) if dy or dx)


def resolve_zbuf(w: Warp, layer_fg: bool, window: int):
    """Splat policy + FG cull + crack median (synthesis.py:207-222, 90-125).

    Returns (zbuf f64 with inf = uncovered, winner int64 (-1 none/crack),
    stage u8).
    """
    H, W = w.shape
    r = w.r
    cen = w.canvas[r:r + H, r:r + W]
    ring = np.full((H, W), KEY_EMPTY, dtype=np.uint64)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            if dy or dx:
                ring = np.minimum(ring, w.canvas[r + dy:r + dy + H, r + dx:r + dx + W])
    center_cov = cen != KEY_EMPTY
    win = np.where(center_cov, cen, ring)
    stage = np.where(center_cov, STAGE_CENTER,
                     np.where(ring != KEY_EMPTY, STAGE_SPLAT, STAGE_NONE)).astype(np.uint8)
    if layer_fg:
        kill = (stage == STAGE_SPLAT) & (_count8(center_cov) < 5)
        win = np.where(kill, KEY_EMPTY, win)
        stage[kill] = STAGE_NONE
    has = win != KEY_EMPTY
    winner = np.where(has, (win & np.uint64((1 << w.b) - 1)).astype(np.int64), -1)
    zbuf = np.full((H, W), np.inf)
    zbuf[has] = w.z_src[winner[has]]

    # crack median over the (window^2 - 1) ring, zero padded (synthesis.py:90-125)
    rc = window // 2
    valid = np.isfinite(zbuf)
    holes = ~valid
    if holes.any() and rc > 0:
        zv = np.where(valid, zbuf, 0.0)
        vals, cnts = [], np.zeros((H, W), dtype=np.int32)
        for dy in range(-rc, rc + 1):
            for dx in range(-rc, rc + 1):
                if dy or dx:
                    nbv = shift2d(valid, dy, dx)
                    vals.append(np.where(nbv, shift2d(zv, dy, dx), np.nan))
                    cnts += nbv
        fill = holes & (cnts >= (window * window) // 2 + 1)
        if fill.any():
            stack = np.stack(vals)[:, fill]
            srt = np.sort(stack, axis=0)       # NaNs sort last
            n = cnts[fill]
            col = np.arange(n.size)
            lo = srt[(n - 1) // 2, col]
            hi = srt[n // 2, col]
            med = np.where(n % 2 == 1, lo, (lo + hi) / 2)
            zbuf[fill] = med
            stage[fill] = STAGE_CRACK
    return zbuf, winner, stage


# ----------------------------------------------------------------------------
# K3: backward colour fetch, mixing, compositing


def backward_fetch(zbuf, src, dst, rgb, color_valid):
    """Stage 3 of warp_layer + ``_bilinear_fetch`` (synthesis.py:224-247, 128-159).

    Returns (colour (H,W,3) f64, valid (H,W) bool).
    """
    src, dst = _cam(src), _cam(dst)
    H, W = zbuf.shape
    out_c = np.zeros((H, W, 3))
    out_v = np.zeros((H, W), dtype=bool)
    vs_i, us_i = np.nonzero(np.isfinite(zbuf))
    if us_i.size == 0:
        return out_c, out_v
    zc = zbuf[vs_i, us_i]
    x, y, z = transfer(zc, dst, src, us_i, vs_i)
    u, v = project(x, y, z, src)
    front = z > 0
    vs_i, us_i, u, v = vs_i[front], us_i[front], u[front], v[front]
    Ws, Hs = src.width, src.height
    inb = (u >= -0.5) & (u <= Ws - 0.5) & (v >= -0.5) & (v <= Hs - 0.5)
    uc = np.clip(u, 0, Ws - 1)
    vc = np.clip(v, 0, Hs - 1)
    u0 = np.floor(uc).astype(np.int64)
    v0 = np.floor(vc).astype(np.int64)
    fu = uc - u0
    fv = vc - v0
    pix = rgb.astype(np.float64)
    col = np.zeros((u.size, 3))
    wsum = np.zeros(u.size)
    for du, dv, wt in ((0, 0, (1 - fu) * (1 - fv)), (1, 0, fu * (1 - fv)),
                       (0, 1, (1 - fu) * fv), (1, 1, fu * fv)):
        uu, vv = u0 + du, v0 + dv
        tin = (uu < Ws) & (vv < Hs)          # uu, vv >= 0 after the clip
        uu, vv = np.minimum(uu, Ws - 1), np.minimum(vv, Hs - 1)
        tw = np.where(tin & color_valid[vv, uu], wt, 0.0)
        col += tw[:, None] * pix[vv, uu]
        wsum += tw
    ok = wsum > 1e-12
    col[ok] /= wsum[ok, None]
    ok &= inb
    out_c[vs_i[ok], us_i[ok]] = col[ok]
    out_v[vs_i[ok], us_i[ok]] = True
    return out_c, out_v


def blend_weight(src, dst, eps: float) -> float:
    """``1/(camera_distance + eps)`` (synthesis.py:249,257; core.py:237-239)."""
    s, d = _cam(src), _cam(dst)
    return 1.0 / (float(np.linalg.norm(s.C - d.C)) + eps)


def warp_layer(rgb, depth, validity, src, dst, cfg, color_valid=None, layer_fg=True):
    """synthesis.warp_layer (synthesis.py:162-258) -> dict of rasters."""
    src, dst = _cam(src), _cam(dst)
    vmask = validity == VALID
    if color_valid is None:
        color_valid = vmask
    w = forward_warp(depth, vmask, src, dst, cfg["splat_radius"])
    zbuf, winner, stage = resolve_zbuf(w, layer_fg, cfg["crack_fill_window"])
    color, valid = backward_fetch(zbuf, src, dst, rgb, color_valid)
    return dict(color=color, depth=np.where(valid, zbuf, 0.0), valid=valid,
                weight=blend_weight(src, dst, cfg["mixing_epsilon"]), winner=winner,
                stage=stage, zbuf=zbuf, camera_id=src.id, layer="fg" if layer_fg else "bg")


def mix_layer(contribs, cfg):
    """synthesis.mix_layer (synthesis.py:261-292)."""
    if not contribs:
        raise ValueError("need at least one contribution")
    shape = contribs[0]["valid"].shape
    z_min = np.full(shape, np.inf)
    for c in contribs:
        z_min = np.where(c["valid"] & (c["depth"] < z_min), c["depth"], z_min)
    thr = z_min + cfg["depth_band_rel"] * z_min
    cacc = np.zeros(shape + (3,))
    dacc = np.zeros(shape)
    wacc = np.zeros(shape)
    for c in contribs:
        wt = np.where(c["valid"] & (c["depth"] <= thr), c["weight"], 0.0)
        cacc += wt[..., None] * c["color"]
        dacc += wt * c["depth"]
        wacc += wt
    valid = wacc > 0
    color = np.zeros_like(cacc)
    depth = np.zeros_like(dacc)
    color[valid] = cacc[valid] / wacc[valid, None]
    depth[valid] = dacc[valid] / wacc[valid]
    return dict(color=color, depth=depth, valid=valid)


def composite(fg, bg, cfg):
    """synthesis.composite (synthesis.py:295-318) -> (rgb u8, provenance u8)."""
    H, W = fg["valid"].shape
    out = np.empty((H, W, 3))
    out[:] = np.asarray(cfg["hole_color"], dtype=np.float64)
    out[bg["valid"]] = bg["color"][bg["valid"]]
    out[fg["valid"]] = fg["color"][fg["valid"]]
    rgb = np.clip(np.rint(out), 0, 255).astype(np.uint8)
    prov = np.zeros((H, W), dtype=np.uint8)
    prov[bg["valid"]] = 1
    prov[fg["valid"]] = 2
    return rgb, prov


DEFAULT_CFG = dict(splat_radius=1, crack_fill_window=3, mixing_epsilon=0.01,
                   depth_band_rel=0.02, hole_color=(0, 0, 0))


def synthesize_view(virtual, refs, cfg=None, debug=False):
    """synthesis.synthesize_view (synthesis.py:331-362).

    ``refs`` is a list of dicts with keys ``calib``, ``rgb`` (H,W,3 u8),
    ``live_depth`` (f32), ``live_validity`` (u8), ``bg_depth`` (f32),
    ``bg_validity`` (u8), in reference order.
    """
    cfg = dict(DEFAULT_CFG, **(cfg or {}))
    if not refs:
        raise ValueError("need at least one reference camera")
    dst = _cam(virtual)
    fgc, bgc = [], []
    for s in refs:
        src = _cam(s["calib"])
        fgc.append(warp_layer(s["rgb"], s["live_depth"], s["live_validity"], src, dst, cfg))
        bgc.append(warp_layer(s["rgb"], s["bg_depth"], s["bg_validity"], src, dst, cfg,
                              color_valid=s["live_validity"] == BACKGROUND, layer_fg=False))
    fg = mix_layer(fgc, cfg)
    bg = mix_layer(bgc, cfg)
    rgb, prov = composite(fg, bg, cfg)
    if debug:
        return rgb, prov, dict(fg_contributions=fgc, bg_contributions=bgc, fg=fg, bg=bg)
    return rgb, prov


def es_view(virtual, frames, cfg=None, hole_closing=True, debug=False):
    """The edge-server path for one view (pipeline.py:514-547).

    ``frames``: list of dicts with ``calib``, ``rgb``, ``mm`` (u16),
    ``validity`` (u8 sidecar), ``bg_depth``, ``bg_validity``. Runs the mm
    decode, the bilateral hole fill and the synthesis, in that order.
    """
    refs = []
    for f in frames:
        d, v = decode_mm(f["mm"], f["validity"])
        if hole_closing:
            d, v, _ = bilateral_close_holes(d, v, f["rgb"])
        refs.append(dict(calib=f["calib"], rgb=f["rgb"], live_depth=d, live_validity=v,
                         bg_depth=f["bg_depth"], bg_validity=f["bg_validity"]))
    return synthesize_view(virtual, refs, cfg, debug=debug)


# ----------------------------------------------------------------------------
# capture-server chain


def correct_depth(depth, validity, alpha, beta):
    """depthproc.correct_depth (depthproc.py:67-84)."""
    d = depth.astype(np.float64).copy()
    val = validity.copy()
    ok = val == VALID
    z = d[ok]
    d[ok] = (alpha * z + beta) * z
    val[ok & (d <= 0)] = INVALID
    d[val != VALID] = 0.0
    return d.astype(np.float32), val


def bg_train(mean, var, rgb, first, rho=0.02, var_floor=4.0):
    """depthproc.bg_train (depthproc.py:121-136), in place on mean/var."""
    x = rgb.astype(np.float64)
    if first:
        mean[:] = x
        var[:] = var_floor
    else:
        mean[:] = (1.0 - rho) * mean + rho * x
        var[:] = np.maximum((1.0 - rho) * var + rho * (x - mean) ** 2, var_floor)


def classify_fg(mean, var, rgb, threshold=3.5):
    """depthproc.classify_fg (depthproc.py:139-149)."""
    x = rgb.astype(np.float64)
    return np.sum((x - mean) ** 2 / var, axis=-1) > threshold ** 2


def remove_bg_depth(depth, validity, fg_mask):
    """depthproc.remove_bg_depth (depthproc.py:152-164)."""
    val = validity.copy()
    d = depth.copy()
    bg = ~np.asarray(fg_mask, dtype=bool)
    val[bg] = BACKGROUND
    d[bg] = 0.0
    return d, val


# ---------------------------------------------------------------------------
# MED + Golomb-Rice plane codec (depthcodec.py:281-409), numpy restatement


def med_residuals(x: np.ndarray) -> np.ndarray:
    """``_med_residuals_py`` (depthcodec.py:281-298): x - MED(a left, b up,
    c up-left), zero outside the plane, as int32 (vectorised: the predictor
    reads only the input plane)."""
    x = x.astype(np.int32)
    a = np.zeros_like(x)
    b = np.zeros_like(x)
    c = np.zeros_like(x)
    a[:, 1:] = x[:, :-1]
    b[1:, :] = x[:-1, :]
    c[1:, 1:] = x[:-1, :-1]
    mx, mn = np.maximum(a, b), np.minimum(a, b)
    p = np.where(c >= mx, mn, np.where(c <= mn, mx, a + b - c))
    return x - p


def med_reconstruct(r: np.ndarray) -> np.ndarray:
    """``_med_reconstruct_py`` (depthcodec.py:301-316): the inverse recurrence,
    row by row (int64 running values; the caller casts to uint8)."""
    h, w = r.shape
    x = np.zeros((h, w), np.int64)
    for i in range(h):
        up = x[i - 1] if i > 0 else np.zeros(w, np.int64)
        left = 0
        for j in range(w):
            a = left if j > 0 else 0
            b = int(up[j])
            c = int(up[j - 1]) if (i > 0 and j > 0) else 0
            mx, mn = (a, b) if a > b else (b, a)
            p = mn if c >= mx else (mx if c <= mn else a + b - c)
            left = int(r[i, j]) + p
            x[i, j] = left
    return x


def zigzag(r: np.ndarray) -> np.ndarray:
    return np.where(r >= 0, 2 * r.astype(np.int64), -2 * r.astype(np.int64) - 1)


def rice_k(zz: np.ndarray) -> int:
    """depthcodec.py:380-381: the k of min over (cost, k), k in 0..14."""
    return min((int(np.sum((zz >> k) + 1 + k)), k) for k in range(15))[1]


def rice_encode(zz: np.ndarray, k: int) -> bytes:
    """``_rice_encode_py`` (depthcodec.py:319-334): q zeros, a one, k bits
    MSB-first; vectorised over symbols with a cumulative bit offset."""
    zz = np.asarray(zz, np.int64).ravel()
    q = zz >> k
    lens = q + 1 + k
    off = np.concatenate([[0], np.cumsum(lens)[:-1]]) if zz.size else np.zeros(0, np.int64)
    nbits = int(lens.sum())
    bits = np.zeros(nbits, np.uint8)
    one = off + q
    bits[one] = 1
    for bi in range(k):
        bits[one + 1 + bi] = (zz >> (k - 1 - bi)) & 1
    return np.packbits(bits).tobytes()


def rice_decode(buf: bytes, n: int, k: int):
    """``_rice_decode_py`` (depthcodec.py:337-355): (symbols, ok)."""
    bits = np.unpackbits(np.frombuffer(buf, np.uint8))
    nbits = bits.size
    ones = np.flatnonzero(bits)
    zz = np.zeros(n, np.int64)
    pos = 0
    for s in range(n):
        i = np.searchsorted(ones, pos)
        if i >= ones.size:
            return zz, False
        t = int(ones[i])
        if t + 1 + k > nbits:
            return zz, False
        rem = 0
        for b in bits[t + 1:t + 1 + k]:
            rem = (rem << 1) | int(b)
        zz[s] = ((t - pos) << k) | rem
        pos = t + 1 + k
    return zz, True


def compress_plane(plane: np.ndarray) -> bytes:
    """``_compress_plane`` (depthcodec.py:373-383)."""
    import struct
    import zlib

    zz = zigzag(med_residuals(plane)).ravel()
    k = rice_k(zz)
    stream = rice_encode(zz, k)
    deflated = zlib.compress(stream, 6)
    blob, flag = (deflated, 1) if len(deflated) < len(stream) else (stream, 0)
    return struct.pack(">BBIII", k, flag, zz.size, len(blob),
                       zlib.adler32(np.ascontiguousarray(plane, np.uint8).tobytes())) + blob


def decompress_plane(data: bytes, offset: int, shape):
    """``_decompress_plane`` (depthcodec.py:386-409); raises ValueError."""
    import struct
    import zlib

    k, flag, n, blen, check = struct.unpack_from(">BBIII", data, offset)
    offset += 14
    blob = data[offset:offset + blen]
    if len(blob) != blen:
        raise ValueError("plane blob truncated")
    offset += blen
    stream = zlib.decompress(blob) if flag else blob
    if n != shape[0] * shape[1]:
        raise ValueError("plane symbol count mismatch")
    zz, ok = rice_decode(stream, n, k)
    if not ok:
        raise ValueError("rice stream truncated")
    r = np.where(zz % 2 == 0, zz // 2, -(zz + 1) // 2).astype(np.int32)
    x = med_reconstruct(r.reshape(shape)).astype(np.uint8)
    if zlib.adler32(x.tobytes()) != check:
        raise ValueError("plane checksum mismatch")
    return x, offset


def encode_lossless_payload(y, u, v) -> bytes:
    """encode_lossless's CODEC_PRED_RICE payload (depthcodec.py:437-438)."""
    return b"".join(compress_plane(p) for p in (y, u, v))


# ---------------------------------------------------------------------------
# MVD disk container rasters (mvdio.py, core.py)


def depth_to_millimeters(depth: np.ndarray, validity: np.ndarray) -> np.ndarray:
    """core.py:246-255 (``encode_mm`` above, with f32 input): Valid pixels ->
    clip(round(f32 depth * 1000), 1, 65535) (the product stays float32 under
    numpy 2's promotion of the Python scalar; np.round is half-to-even);
    every other pixel 0."""
    return encode_mm(np.asarray(depth, dtype=np.float32), np.asarray(validity))


def rle_encode(flat: np.ndarray):
    """mvdio.py:34-40: [[code, run], ...] over the flattened raster; a run
    starts at 0 and wherever a value differs from its predecessor."""
    flat = np.asarray(flat).ravel()
    if flat.size == 0:
        return []
    starts = np.concatenate([[0], np.flatnonzero(flat[1:] != flat[:-1]) + 1])
    ends = np.concatenate([starts[1:], [flat.size]])
    return [[int(flat[a]), int(b - a)] for a, b in zip(starts, ends)]


def rle_decode(runs, size: int) -> np.ndarray:
    """mvdio.py:43-52: the runs must cover exactly ``size`` pixels."""
    out = np.empty(size, dtype=np.uint8)
    pos = 0
    for code, n in runs:
        out[pos:pos + n] = code
        pos += n
    if pos != size:
        raise ValueError(f"RLE covers {pos} pixels, expected {size}")
    return out

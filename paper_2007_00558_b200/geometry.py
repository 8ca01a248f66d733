"""Rig API kept on the host: pinhole helpers, camera arcs, rig files.

Mirrors the reference's host-side geometry surface so a user of
``fvv.core``/``fvv.scenegen`` finds the same calls:

* ``project_points`` / ``pixel_rays`` / ``unproject_map`` / ``camera_distance``
  (``core.py:160-239``);
* ``look_at_pose`` / ``arc_pose`` / ``build_camera_arc`` (``scenegen.py:161-223``);
* ``save_rig`` / ``load_rig`` JSON rig files (``core.py:275-328``).

None of this is on the per-pixel path: the per-pixel geometry runs inside the
sm_100a kernels (``csrc/fvv_kernels.cu``). These helpers exist for rig set-up,
tests and selection.
"""

from __future__ import annotations

import json
import math
from pathlib import Path
from typing import Sequence

import numpy as np

from .types import CameraCalibration, CameraIntrinsics, CameraPose

RIG_FORMAT_VERSION = 1


def world_to_camera(points: np.ndarray, pose) -> np.ndarray:
    return (np.asarray(points, dtype=np.float64) - pose.center) @ pose.rotation.T


def camera_to_world(points: np.ndarray, pose) -> np.ndarray:
    return np.asarray(points, dtype=np.float64) @ pose.rotation + pose.center


def project_points(points: np.ndarray, calib):
    """(N,3) world points -> (uv, z, in_front), ``core.py:199-214``."""
    p = world_to_camera(points, calib.pose)
    z = p[..., 2]
    k = calib.intrinsics
    with np.errstate(divide="ignore", invalid="ignore"):
        u = k.fx * p[..., 0] / z + k.cx
        v = k.fy * p[..., 1] / z + k.cy
    return np.stack([u, v], axis=-1), z, z > 0


def pixel_rays(calib) -> np.ndarray:
    """(H, W, 3) camera-frame rays with z = 1, ``core.py:217-227``."""
    k = calib.intrinsics
    xs = (np.arange(k.width, dtype=np.float64) - k.cx) / k.fx
    ys = (np.arange(k.height, dtype=np.float64) - k.cy) / k.fy
    out = np.ones((k.height, k.width, 3))
    out[..., 0] = xs[None, :]
    out[..., 1] = ys[:, None]
    return out


def unproject_map(depth: np.ndarray, calib) -> np.ndarray:
    return camera_to_world(pixel_rays(calib) * np.asarray(depth, np.float64)[..., None],
                           calib.pose)


def camera_distance(a, b) -> float:
    """Distance between camera centres in metres (``core.py:237-239``).

    Evaluated with the same numpy expression as the reference so the blend
    weight ``1/(d + eps)`` handed to the kernels is bit-identical.
    """
    return float(np.linalg.norm(a.center - b.center))


def look_at_pose(center, target) -> CameraPose:
    """Pose at ``center`` looking at ``target``; world +y is down.

    Same construction as ``scenegen.look_at_pose`` (``scenegen.py:208-223``):
    x = down × forward, y = forward × x. A vertical optical axis is rejected.
    """
    c = np.asarray(center, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - c
    n = np.linalg.norm(fwd)
    if n == 0:
        raise ValueError("camera center and look-at target coincide")
    zax = fwd / n
    xax = np.cross(np.array([0.0, 1.0, 0.0]), zax)
    nx = np.linalg.norm(xax)
    if nx < 1e-12:
        raise ValueError("optical axis may not be vertical")
    xax = xax / nx
    yax = np.cross(zax, xax)
    return CameraPose(rotation=np.stack([xax, yax, zax]), center=c)


def arc_pose(radius: float, phi: float, height: float = 0.0) -> CameraPose:
    """Pose on a circle of ``radius`` around the origin at angle ``phi``.

    ``phi = 0`` sits on -z looking toward +z (``scenegen.py:202-205``);
    ``height`` is a world-y offset (+y is down), the look-at target stays on
    the arc axis at the same height so the optical axis remains horizontal.
    """
    c = np.array([radius * math.sin(phi), height, -radius * math.cos(phi)])
    return look_at_pose(c, np.array([0.0, height, 0.0]))


def build_camera_arc(n: int, spacing: float, span_deg: float, *, width: int = 160,
                     height: int = 120, hfov_deg: float = 60.0) -> list:
    """``n`` cameras on an arc with chord ``spacing`` (``scenegen.py:161-199``)."""
    if n < 2:
        raise ValueError("need at least 2 cameras")
    if spacing <= 0:
        raise ValueError("spacing must be positive")
    if not (0 < span_deg < 180):
        raise ValueError("span must be in (0, 180) degrees")
    gap = math.radians(span_deg) / (n - 1)
    radius = spacing / (2.0 * math.sin(gap / 2.0))
    f = (width / 2.0) / math.tan(math.radians(hfov_deg) / 2.0)
    intr = CameraIntrinsics(f, f, width / 2.0, height / 2.0, width, height)
    return [CameraCalibration(i, intr, arc_pose(radius, (i - (n - 1) / 2.0) * gap))
            for i in range(n)]


def arc_rig(n: int, radius: float, gap_deg: float, intr: CameraIntrinsics,
            height: float = 0.0, first_id: int = 0) -> list:
    """Cameras on a radius-``radius`` arc, ``gap_deg`` apart, centred on phi=0.

    This is the parameterisation BASELINE.json's configs are quoted in
    ("3 m-radius arc spanning 80 degrees, 10 degrees apart").
    """
    gap = math.radians(gap_deg)
    return [CameraCalibration(first_id + i, intr,
                              arc_pose(radius, (i - (n - 1) / 2.0) * gap, height))
            for i in range(n)]


def save_rig(path, rig: Sequence) -> None:
    """JSON rig file with the reference's field list (``core.py:278-297``)."""
    cams = []
    for c in rig:
        k = c.intrinsics
        cams.append(dict(id=int(c.id), fx=float(k.fx), fy=float(k.fy), cx=float(k.cx),
                         cy=float(k.cy), width=int(k.width), height=int(k.height),
                         rotation=[float(x) for x in np.ravel(c.pose.rotation)],
                         center=[float(x) for x in c.pose.center]))
    Path(path).write_text(json.dumps({"version": RIG_FORMAT_VERSION, "cameras": cams},
                                     indent=2))


def load_rig(path) -> list:
    doc = json.loads(Path(path).read_text())
    if doc.get("version") != RIG_FORMAT_VERSION:
        raise ValueError(f"unsupported rig file version {doc.get('version')!r}")
    out, seen = [], set()
    for e in doc["cameras"]:
        cid = int(e["id"])
        if cid in seen:
            raise ValueError(f"duplicate camera id {cid} in rig file")
        seen.add(cid)
        intr = CameraIntrinsics(float(e["fx"]), float(e["fy"]), float(e["cx"]),
                                float(e["cy"]), int(e["width"]), int(e["height"]))
        pose = CameraPose(np.array(e["rotation"], dtype=np.float64).reshape(3, 3),
                          np.array(e["center"], dtype=np.float64))
        out.append(CameraCalibration(cid, intr, pose))
    return out

"""Value types of the view-synthesis boundary.

Names, fields, validation rules and error behaviour follow the reference's
``fvv.core`` value types (``/root/reference/pkg/src/fvv/core.py:28-153``) so
objects built by either package can be passed to the other (duck typing on
``.intrinsics``/``.pose``/``.pixels``/``.depth``/``.validity``).

Conventions (``core.py:3-10``): top-left image origin, pixel centres at
integer coordinates, ``p_cam = R (X - C)``, camera y down / z forward,
depth = camera-frame z in metres.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np

ORTHONORMAL_TOL = 1e-9


class Validity(IntEnum):
    """Per-pixel depth flag stored as uint8 (``core.py:28-33``)."""

    VALID = 0
    INVALID = 1
    BACKGROUND = 2


@dataclass(frozen=True)
class CameraIntrinsics:
    """Pinhole intrinsics (``core.py:36-57``); even sizes for YUV420."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if not (self.fx > 0 and self.fy > 0):
            raise ValueError(f"focal lengths must be positive, got ({self.fx}, {self.fy})")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point must lie inside the image")
        if self.width % 2 or self.height % 2:
            raise ValueError(f"width and height must be even, got {self.width}x{self.height}")

    def matrix(self) -> np.ndarray:
        k = np.eye(3)
        k[0, 0], k[1, 1], k[0, 2], k[1, 2] = self.fx, self.fy, self.cx, self.cy
        return k


@dataclass(frozen=True)
class CameraPose:
    """World->camera rotation plus camera centre (``core.py:60-79``)."""

    rotation: np.ndarray
    center: np.ndarray

    def __post_init__(self):
        r = np.asarray(self.rotation, dtype=np.float64)
        c = np.asarray(self.center, dtype=np.float64)
        if r.shape != (3, 3):
            raise ValueError(f"rotation must be 3x3, got {r.shape}")
        if c.shape != (3,):
            raise ValueError(f"center must be a 3-vector, got {c.shape}")
        if not (np.isfinite(r).all() and np.isfinite(c).all()):
            raise ValueError("pose contains non-finite values")
        if np.abs(r.T @ r - np.eye(3)).max() > ORTHONORMAL_TOL:
            raise ValueError("rotation is not orthonormal")
        if abs(np.linalg.det(r) - 1.0) > ORTHONORMAL_TOL:
            raise ValueError("rotation must have determinant +1")
        object.__setattr__(self, "rotation", r)
        object.__setattr__(self, "center", c)


@dataclass(frozen=True)
class CameraCalibration:
    id: int
    intrinsics: CameraIntrinsics
    pose: CameraPose


@dataclass(frozen=True)
class ColorFrame:
    """uint8 RGB raster (``core.py:89-102``)."""

    width: int
    height: int
    pixels: np.ndarray
    timestamp_us: int = 0

    def __post_init__(self):
        px = np.asarray(self.pixels, dtype=np.uint8)
        if px.shape != (self.height, self.width, 3):
            raise ValueError(
                f"pixel raster shape {px.shape} does not match {self.height}x{self.width}x3")
        object.__setattr__(self, "pixels", px)


@dataclass(frozen=True)
class DepthFrame:
    """float32 metric depth + uint8 validity (``core.py:105-130``).

    Valid pixels must carry positive finite depth.
    """

    width: int
    height: int
    depth: np.ndarray
    validity: np.ndarray
    timestamp_us: int = 0

    def __post_init__(self):
        d = np.asarray(self.depth, dtype=np.float32)
        v = np.asarray(self.validity, dtype=np.uint8)
        if d.shape != (self.height, self.width):
            raise ValueError(f"depth shape {d.shape} does not match {self.height}x{self.width}")
        if v.shape != d.shape:
            raise ValueError("validity shape does not match depth shape")
        dv = d[v == Validity.VALID]
        if dv.size and not (np.isfinite(dv).all() and (dv > 0).all()):
            raise ValueError("Valid pixels must carry positive finite depth")
        object.__setattr__(self, "depth", d)
        object.__setattr__(self, "validity", v)

    @property
    def valid_mask(self) -> np.ndarray:
        return self.validity == Validity.VALID


@dataclass(frozen=True)
class MvdFrame:
    """Colour + depth of one camera at one instant (``core.py:133-143``)."""

    camera_id: int
    color: ColorFrame
    depth: DepthFrame

    @property
    def timestamp_us(self) -> int:
        return self.color.timestamp_us


@dataclass(frozen=True)
class DepthRange:
    z_near: float
    z_far: float

    def __post_init__(self):
        if not (0 < self.z_near < self.z_far):
            raise ValueError(f"need 0 < z_near < z_far, got ({self.z_near}, {self.z_far})")

"""Pinhole camera and Gaussian primitive (host side).

Mirrors reference ``pkg/src/nexsplat/primitives.py:96-209``.  The camera is
a handful of doubles handed to the kernels through the C-ABI ``nxs_camera``
struct; nothing per-pixel is materialised on the host (the kernels derive
the pixel rays of reference ``Camera.pixel_directions``, primitives.py:192-203,
on the fly).  ``pixel_directions`` is kept for API parity.

Any object with ``position, rotation, focal, cx, cy, width, height``
attributes (for example the reference's own ``nexsplat.Camera``) is
accepted by the render entry points.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Camera",
    "GaussianPrimitive",
    "quat_to_rot",
    "SH_C0",
    "SH_C1",
    "ALPHA_EPS",
    "ALPHA_MAX",
    "OPACITY_MIN",
    "SCALE_MIN",
    "NEAR_PLANE",
    "DEFAULT_ALPHA_CUTOFF",
    "DEFAULT_MAX_SAMPLES",
]

# reference primitives.py:35-42 and compositor.py:29-33
OPACITY_MIN = 1e-4
SCALE_MIN = 1e-6
NEAR_PLANE = 1e-4
DEFAULT_ALPHA_CUTOFF = 1.0 / 255.0
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
ALPHA_EPS = 1e-6
ALPHA_MAX = 1.0 - ALPHA_EPS
DEFAULT_MAX_SAMPLES = 128


def quat_to_rot(q: np.ndarray) -> np.ndarray:
    """Rotation matrices from (w, x, y, z) quaternions, normalised
    internally (reference primitives.py:45-64)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


@dataclass
class GaussianPrimitive:
    """One splat (reference primitives.py:96-137), same validation."""

    center: np.ndarray
    scale: np.ndarray
    rotation: np.ndarray
    opacity: float
    sh: np.ndarray

    def __post_init__(self) -> None:
        self.center = np.asarray(self.center, dtype=np.float64).reshape(3)
        self.scale = np.asarray(self.scale, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(4)
        self.sh = np.atleast_2d(np.asarray(self.sh, dtype=np.float64))
        if self.sh.shape not in ((3, 1), (3, 4)):
            raise ValueError(f"sh must have shape (3,1) or (3,4), got {self.sh.shape}")
        if np.any(self.scale < SCALE_MIN):
            raise ValueError(f"scale components must be >= {SCALE_MIN}")
        norm = np.linalg.norm(self.rotation)
        if abs(norm - 1.0) > 1e-9:
            raise ValueError(f"rotation quaternion must be unit length, |q| = {norm}")
        if not 0.0 < self.opacity <= 1.0:
            raise ValueError(f"opacity must be in (0, 1], got {self.opacity}")
        self.opacity = float(np.clip(self.opacity, OPACITY_MIN, ALPHA_MAX))


@dataclass
class Camera:
    """Pinhole camera; ``rotation`` maps camera axes (right, down, forward)
    to world axes (reference primitives.py:153-209)."""

    position: np.ndarray
    rotation: np.ndarray
    focal: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self) -> None:
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        if self.focal <= 0 or self.width <= 0 or self.height <= 0:
            raise ValueError("focal length and image dimensions must be positive")

    @classmethod
    def from_look_at(cls, position, look_at, up, fov_deg: float,
                     width: int, height: int) -> "Camera":
        position = np.asarray(position, dtype=np.float64)
        forward = np.asarray(look_at, dtype=np.float64) - position
        fn = np.linalg.norm(forward)
        if fn == 0:
            raise ValueError("camera position and look-at point coincide")
        forward = forward / fn
        upv = np.asarray(up, dtype=np.float64)
        right = np.cross(forward, upv)
        rn = np.linalg.norm(right)
        if rn < 1e-12:
            raise ValueError("up vector is parallel to the view direction")
        right = right / rn
        down = np.cross(forward, right)
        R = np.stack([right, down, forward], axis=1)
        focal = 0.5 * width / np.tan(np.radians(fov_deg) / 2.0)
        return cls(position, R, focal, width / 2.0, height / 2.0, width, height)

    def pixel_directions(self) -> np.ndarray:
        """Unit world directions through all pixel centres, (H, W, 3)."""
        j = np.arange(self.width) + 0.5
        i = np.arange(self.height) + 0.5
        d_cam = np.empty((self.height, self.width, 3))
        d_cam[..., 0] = ((j - self.cx) / self.focal)[None, :]
        d_cam[..., 1] = ((i - self.cy) / self.focal)[:, None]
        d_cam[..., 2] = 1.0
        d_world = d_cam @ self.rotation.T
        return d_world / np.linalg.norm(d_world, axis=-1, keepdims=True)

"""Synthetic benchmark workloads.

The canonical scene generalises reference ``studies.py:170-181``
(``dense_scene``) with the band-1 SH draw of ``studies.py:142-143`` and a
density-preserving scale factor (5000/n)^(1/3); parameters are rounded to
float32 (the device precision) so a float64 consumer sees identical inputs.
Views: ``Camera.from_look_at(pos, (0,0,3.5), (0,1,0), 55°, W, H)`` with
view v of V at pos = 0.4·(cos 2πv/V, sin 2πv/V, 0); adjoint seeds
U(0.2, 1) from ``default_rng(1000 + v)``.
"""
from __future__ import annotations

import numpy as np

from .camera import SH_C0, Camera
from .render import SceneArrays

__all__ = ["canonical_scene", "canonical_camera", "canonical_seed", "CONFIGS"]

# BASELINE.json configs (C1..C5)
CONFIGS = {
    "C1": dict(n=1_000, width=64, height=64, views=1, model="exponential"),
    "C2": dict(n=100_000, width=512, height=512, views=1, model="softplus"),
    "C3": dict(n=1_000_000, width=1920, height=1080, views=1, model="softplus"),
    "C4": dict(n=1_000_000, width=1920, height=1080, views=64, model="softplus"),
    "C5": dict(n=5_000_000, width=3840, height=2160, views=256, model="blended"),
}


def canonical_scene(n: int, seed: int = 5, sh_coeffs: int = 4) -> SceneArrays:
    rng = np.random.default_rng(seed)
    s = (5000.0 / n) ** (1.0 / 3.0)
    centers = np.column_stack([rng.uniform(-1.6, 1.6, n), rng.uniform(-1.6, 1.6, n),
                               rng.uniform(2.0, 8.0, n)])
    scales = rng.uniform(0.05, 0.18, (n, 3)) * s
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opac = rng.uniform(0.3, 0.9, n)
    sh = np.zeros((n, 3, sh_coeffs))
    sh[:, :, 0] = rng.uniform(0.2, 1.0, (n, 3)) / SH_C0
    if sh_coeffs == 4:
        sh[:, :, 1:] = rng.normal(0.0, 0.15, (n, 3, 3))
    f = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
    return SceneArrays(f(centers), f(scales), f(quats), f(opac), f(sh))


def canonical_camera(width: int, height: int, view: int = 0, n_views: int = 1) -> Camera:
    if n_views <= 1:
        pos = [0.0, 0.0, 0.0]
    else:
        a = 2.0 * np.pi * view / n_views
        pos = [0.4 * np.cos(a), 0.4 * np.sin(a), 0.0]
    return Camera.from_look_at(pos, [0.0, 0.0, 3.5], [0.0, 1.0, 0.0], 55.0, width, height)


def canonical_seed(width: int, height: int, view: int = 0) -> np.ndarray:
    return np.random.default_rng(1000 + view).uniform(0.2, 1.0, (height, width, 3))

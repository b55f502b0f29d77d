"""Shared test helpers: golden-fixture loading and the parity protocol
(SURVEY §8c): identical fp32-rounded inputs, decision-margin masks,
tolerance |x - ref| <= 1e-6 + 1e-5|ref| (BASELINE north_star), and the
mass-scaled gradient bound |g - ref| <= 1e-6 + 1e-5 S."""
from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
RTOL, ATOL = 1e-5, 1e-6
GRAD_FIELDS = ("centers", "scales", "quats", "opacities", "sh")


class Cam:
    def __init__(self, position, rotation, focal, cx, cy, width, height):
        self.position = np.asarray(position, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(rotation, dtype=np.float64).reshape(3, 3)
        self.focal, self.cx, self.cy = float(focal), float(cx), float(cy)
        self.width, self.height = int(width), int(height)


class Arrs:
    def __init__(self, centers, scales, quats, opacities, sh):
        self.centers, self.scales, self.quats = centers, scales, quats
        self.opacities, self.sh = opacities, sh

    def __len__(self):
        return len(self.opacities)


class Model:
    def __init__(self, variant, param=0.0):
        self.variant, self.param = variant, float(param)


MODELS = {
    "exponential": Model("exponential"),
    "linear": Model("linear"),
    "quadratic_0.5": Model("quadratic", 0.5),
    "softplus_20": Model("softplus", 20.0),
    "blended_0.5": Model("blended", 0.5),
    "vicini_0.3": Model("vicini", 0.3),
    "power_law_2": Model("power_law", 2.0),
}


def load(name):
    return dict(np.load(GOLDEN / name))


def cam_from(d, prefix="cam_"):
    return Cam(d[prefix + "position"], d[prefix + "rotation"], d[prefix + "focal"],
               d[prefix + "cx"], d[prefix + "cy"], d[prefix + "width"], d[prefix + "height"])


def scene_from(d, prefix="scene_"):
    return Arrs(*(np.asarray(d[prefix + k], dtype=np.float64)
                  for k in ("centers", "scales", "quats", "opacities", "sh")))


def close(x, ref, rtol=RTOL, atol=ATOL):
    return np.abs(np.asarray(x) - np.asarray(ref)) <= atol + rtol * np.abs(ref)


def grad_report(g, ref, mass=None):
    """(strict failures, mass-scaled failures, total entries)."""
    strict = mass_f = total = 0
    for k in GRAD_FIELDS:
        a, b = np.asarray(g[k], dtype=np.float64), np.asarray(ref[k], dtype=np.float64)
        bad = ~close(a, b)
        strict += int(bad.sum())
        total += a.size
        if mass is not None:
            mass_f += int((np.abs(a - b) > ATOL + RTOL * np.asarray(mass[k])).sum())
    return strict, mass_f, total


def exact_depths(centers, cam):
    """View depths (μ - o)·forward in 80-bit extended precision."""
    c = np.asarray(centers, dtype=np.longdouble) - np.asarray(cam.position, dtype=np.longdouble)
    f = np.asarray(cam.rotation, dtype=np.longdouble)[:, 2]
    return (c * f).sum(axis=1)


def assert_order_matches_up_to_ties(got, ref, depths, ulps=4):
    """Orders must agree except between Gaussians whose depths agree to a
    few ulps (the reference's own depth rounding is CPU-dependent)."""
    got, ref = np.asarray(got), np.asarray(ref)
    assert sorted(got.tolist()) == sorted(ref.tolist())
    bad = np.nonzero(got != ref)[0]
    if bad.size == 0:
        return 0
    dg = depths[got[bad]].astype(np.float64)
    dr = depths[ref[bad]].astype(np.float64)
    tol = ulps * np.spacing(np.abs(dr))
    assert (np.abs(dg - dr) <= tol).all(), bad[np.abs(dg - dr) > tol][:10]
    return int(bad.size)

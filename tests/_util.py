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
    """(strict failures, mass-scaled failures, total entries); the mass
    scale is the componentwise one where the oracle provides it."""
    strict = mass_f = total = 0
    for k in GRAD_FIELDS:
        a, b = np.asarray(g[k], dtype=np.float64), np.asarray(ref[k], dtype=np.float64)
        bad = ~close(a, b)
        strict += int(bad.sum())
        total += a.size
        if mass is not None:
            sc = np.asarray(mass.get(k + "_c", mass[k]))
            mass_f += int((np.abs(a - b) > ATOL + RTOL * sc).sum())
    return strict, mass_f, total


def grad_report_full(g, ref, mass, cancel=1e-2):
    """Per-group parity counts.

    strict   : |g - ref| > 1e-6 + 1e-5|ref| (BASELINE north_star)
    strict_nc: the strict failures whose reference is NOT cancellation-
               limited, |ref| >= ``cancel`` x its componentwise scale S_c
               (a sum that kept < 1 % of its terms' magnitude is determined
               only to ~eps·S_c by any fp32 evaluation)
    mass_c   : |g - ref| > 1e-6 + 1e-5 S_c, S_c the componentwise
               absolute-evaluation scale of the oracle (``mass[k + '_c']``,
               SURVEY §8c) — the gate
    mass     : the same with the r01 normwise geometric scale (reported)"""
    rep = {"total": 0, "strict": 0, "strict_nc": 0, "mass": 0, "mass_c": 0, "groups": {}}
    for k in GRAD_FIELDS:
        a, b = np.asarray(g[k], dtype=np.float64), np.asarray(ref[k], dtype=np.float64)
        err = np.abs(a - b)
        sc = np.asarray(mass.get(k + "_c", mass[k]))
        bad = ~close(a, b)
        s = int(bad.sum())
        snc = int((bad & (np.abs(b) >= cancel * sc)).sum())
        mw = int((err > ATOL + RTOL * np.asarray(mass[k])).sum())
        mc = int((err > ATOL + RTOL * sc).sum())
        rep["groups"][k] = {"entries": a.size, "strict": s, "strict_nc": snc, "mass": mw,
                            "mass_c": mc, "nonzero_ref": int((b != 0).sum())}
        rep["total"] += a.size
        rep["strict"] += s
        rep["strict_nc"] += snc
        rep["mass"] += mw
        rep["mass_c"] += mc
    return rep


def strict_budget(ref, basis="entries", frac=1e-3):
    """The strict-failure budget: ``frac`` of the gradient entries (at least
    1).  ``basis="touched"`` counts only the entries the reference touches
    (non-zero) — for sampled-pixel cases, where most of a large scene's
    entries are exact zeros on both sides and would only dilute it."""
    if basis == "touched":
        n = sum(int((np.asarray(ref[k]) != 0).sum()) for k in GRAD_FIELDS)
    else:
        n = sum(np.asarray(ref[k]).size for k in GRAD_FIELDS)
    return max(1, int(frac * n))


def write_report(group, tag, rep):
    """Parity counts of one case -> $NXS_PARITY_DIR/<group>/<tag>.json
    (default gpurun_out/; collected into profiles/ by hand)."""
    import json
    import os
    d = Path(os.environ.get("NXS_PARITY_DIR", GOLDEN.parents[1] / "gpurun_out" / "parity"))
    d = d / group
    try:
        d.mkdir(parents=True, exist_ok=True)
        (d / f"{tag}.json").write_text(json.dumps(rep, indent=1, default=str))
    except OSError:
        pass


def check_grads(group, tag, got, ref, mass, basis="entries", **extra):
    """The north-star gradient bar: every entry inside the componentwise
    mass-scaled bound; strict failures of the non-cancelled entries <= 0.1 %
    of the entries (of the touched entries with ``basis="touched"``).
    Writes the counts."""
    rep = grad_report_full(got, ref, mass)
    rep["strict_budget"] = strict_budget(ref, basis)
    rep["budget_basis"] = basis
    rep.update(extra)
    write_report(group, tag, rep)
    assert rep["mass_c"] == 0, rep
    assert rep["strict_nc"] <= rep["strict_budget"], rep
    return rep


def mask_parts(fwd, model, t_order):
    """(decision-margin mask without t ties, t-tie-only mask) of an oracle
    forward (see splat_oracle.margin_mask)."""
    dec = fwd["amargin"] < 1e-5
    dec = dec | (fwd["sat"] if model.variant == "exponential" else fwd["smargin"] < 1e-5)
    tt = (fwd["tmargin"] < 1e-6) & ~dec if t_order else np.zeros_like(dec)
    return dec, tt


def check_masked(fwd, model, t_order, n, t_cap=0.03):
    """Masked samples: decision margins <= 1 %, all masks <= ``t_cap`` in the
    t-ordered modes (two candidates within 1e-6 relative peak depth)."""
    dec, tt = mask_parts(fwd, model, t_order)
    assert dec.sum() <= max(1, n // 100), (int(dec.sum()), n)
    assert (dec | tt).sum() <= max(1, int(t_cap * n)), (int(dec.sum()), int(tt.sum()), n)
    return int(dec.sum()), int(tt.sum())


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

"""CPU restatement of the reference's per-ray batched compositor (SURVEY §8
row f4) — TEST INFRASTRUCTURE ONLY: the checker for csrc/batch.cu; nothing
in the product imports it.  Pinned against the reference's own outputs
(tests/golden/golden_batch.npz, tests/golden/make_golden.py ``batch``).

Restates, in float64 numpy, a sequential scan per ray:
  composite_batch          reference pkg/src/nexsplat/compositor.py:84-171
  discrete_extinction      transmittance.py:215-265
  finite_diff_gradients    adjoint.py:195-222
"""
from __future__ import annotations

import numpy as np


def extinction(variant, param, a, tau, prod):
    """transmittance.py:232-262 (vectorised over rays)."""
    if variant == "exponential":
        return a * prod
    if variant == "linear":
        return a.copy()
    if variant == "quadratic":
        return a * (1.0 + param * tau)
    if variant == "blended":
        return a * (1.0 - param * (1.0 - prod))
    if variant == "vicini":
        return a + param * (a * prod - a)
    if variant == "power_law":
        if param == -1.0:
            return a.copy()
        if abs(param) < 1e-4:
            return a * np.exp(-tau)
        base = 1.0 + tau * param
        return np.where(base > 0, a * np.where(base > 0, base, 1.0) ** (-(1.0 + param) / param),
                        0.0)
    k = param  # softplus
    x = k * (1.0 - tau)
    sig = np.where(x >= 0, 1.0 / (1.0 + np.exp(-np.abs(x))),
                   np.exp(-np.abs(x)) / (1.0 + np.exp(-np.abs(x))))
    return a * (k / np.logaddexp(0.0, k)) * sig


def composite_batch(variant, param, alpha, emission, background, valid=None):
    alpha = np.asarray(alpha, dtype=np.float64)
    emission = np.asarray(emission, dtype=np.float64)
    bg = np.asarray(background, dtype=np.float64)
    R, N = alpha.shape
    valid = np.ones((R, N), dtype=bool) if valid is None else np.asarray(valid, dtype=bool)
    tau, prod, cum = np.zeros(R), np.ones(R), np.zeros(R)
    k0 = np.full(R, N, dtype=np.int64)
    weights = np.zeros((R, N))
    rad = np.zeros((R, 3))
    sa, sea = np.zeros(R), np.zeros((R, 3))
    e_k = np.broadcast_to(bg, (R, 3)).copy()
    t_k = np.zeros(R)
    for i in range(N):
        v = valid[:, i]
        a = np.where(v, alpha[:, i], 0.0)
        live = k0 == N
        raw = np.where(v, extinction(variant, param, a, tau, prod), 0.0)
        before = cum.copy()
        cum = cum + np.where(live, raw, 0.0)
        sat_now = live & (cum >= 1.0)
        w = np.where(sat_now, 1.0 - before, np.where(live, raw, 0.0))
        weights[:, i] = w
        rad += w[:, None] * emission[:, i]
        tail = live & ~sat_now & v & (i >= 1)
        sa += np.where(tail, a, 0.0)
        sea += np.where(tail, a, 0.0)[:, None] * emission[:, i]
        e_k = np.where(sat_now[:, None], emission[:, i], e_k)
        t_k = np.where(sat_now, w, t_k)
        k0 = np.where(sat_now, i, k0)
        tau += a
        prod *= 1.0 - a
    sat = k0 < N
    residual = np.where(sat, 0.0, 1.0 - cum)
    rad += bg[None, :] * residual[:, None]
    return {"weights": weights, "radiance": rad, "residual": residual,
            "k0": np.where(N == 0, 0, k0),
            "overdraw": np.where(sat, k0 + 1, valid.sum(axis=1)),
            "e_k": e_k, "theta0": sea - e_k * sa[:, None],
            "t_k": np.where(sat, t_k, residual)}


def finite_diff_gradients(variant, param, alpha, emission, background, eps=1e-5,
                          seed=(1.0, 1.0, 1.0)):
    """adjoint.py:195-222: (d_alpha, d_emission)."""
    seed = np.asarray(seed, dtype=np.float64)
    alpha = np.asarray(alpha, dtype=np.float64)
    emission = np.asarray(emission, dtype=np.float64).reshape(-1, 3)
    n = len(alpha)
    rows = 4 * n
    al = np.tile(alpha, (rows, 1))
    em = np.tile(emission, (rows, 1, 1))
    r = np.arange(n)
    al[r, r] += eps
    al[n + r, r] -= eps
    em[2 * n + r, r, :] += eps
    em[3 * n + r, r, :] -= eps
    rad = composite_batch(variant, param, al, em, background)["radiance"]
    d_a = (rad[:n] - rad[n:2 * n]) / (2 * eps)
    d_e = (rad[2 * n:3 * n] - rad[3 * n:]) / (2 * eps)
    return d_a @ seed, d_e * seed[None, :]

"""CPU restatement of the reference's train-step neighbours (SURVEY §8 row
f2) — TEST INFRASTRUCTURE ONLY: the checker for the device loss / Adam
kernels (paper_2603_02887_b200/csrc/train.cu); nothing in the product
imports it.

Pinned against the reference's own outputs (tests/golden/golden_train.npz,
written by tests/golden/make_golden.py ``train``).  Restates, in float64
numpy:
  linear_to_srgb / dsrgb_dlinear   reference pkg/src/nexsplat/images.py:31-50
  _gauss_kernel / _window_filter   optimizer.py:53-65 (scipy correlate1d,
                                   mode "constant" = zero padding)
  ssim (+ gradient)                optimizer.py:75-111
  mse / psnr                       optimizer.py:114-125
  loss                             optimizer.py:128-152
  bounded_adam_step                optimizer.py:173-204
"""
from __future__ import annotations

import numpy as np

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
ADAM_BETA1, ADAM_BETA2, ADAM_EPS = 0.9, 0.999, 1e-8
OPACITY_MIN, SCALE_MIN, ALPHA_MAX = 1e-4, 1e-6, 1.0 - 1e-6
_T, _SLOPE1 = 0.0031308, 1.055 / 2.4


def linear_to_srgb(x):
    """images.py:31-36 (tangent-extended above 1)."""
    x = np.asarray(x, dtype=np.float64)
    mid = 1.055 * np.power(np.clip(x, _T, 1.0), 1.0 / 2.4) - 0.055
    return np.where(x <= _T, 12.92 * x, np.where(x <= 1.0, mid, 1.0 + _SLOPE1 * (x - 1.0)))


def dsrgb_dlinear(x):
    """images.py:47-50."""
    x = np.asarray(x, dtype=np.float64)
    mid = _SLOPE1 * np.power(np.clip(x, _T, 1.0), 1.0 / 2.4 - 1.0)
    return np.where(x <= _T, 12.92, np.where(x <= 1.0, mid, _SLOPE1))


def _kernel():
    r = np.arange(SSIM_WINDOW) - SSIM_WINDOW // 2
    k = np.exp(-0.5 * (r / SSIM_SIGMA) ** 2)
    return k / k.sum()


_K = _kernel()


def _correlate(img, axis):
    """1-D correlation with the window along ``axis``, zero padding."""
    h = SSIM_WINDOW // 2
    img = np.moveaxis(img, axis, 0)
    pad = np.zeros((img.shape[0] + 2 * h,) + img.shape[1:])
    pad[h:h + img.shape[0]] = img
    out = np.zeros_like(img, dtype=np.float64)
    for t in range(SSIM_WINDOW):
        out += _K[t] * pad[t:t + img.shape[0]]
    return np.moveaxis(out, 0, axis)


def window_filter(img):
    """optimizer.py:63-65: rows then columns."""
    return _correlate(_correlate(np.asarray(img, dtype=np.float64), 0), 1)


def ssim(x, y, with_grad=False):
    """optimizer.py:75-111: mean SSIM over fully-interior windows."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError("image shapes differ")
    h, w = x.shape[:2]
    if h < SSIM_WINDOW or w < SSIM_WINDOW:
        raise ValueError("images must be at least 11 pixels on each side")
    half = SSIM_WINDOW // 2
    mask = np.zeros((h, w, 1))
    mask[half:h - half, half:w - half] = 1.0
    mu_x, mu_y = window_filter(x), window_filter(y)
    sxx = window_filter(x * x) - mu_x * mu_x
    syy = window_filter(y * y) - mu_y * mu_y
    sxy = window_filter(x * y) - mu_x * mu_y
    a1 = 2 * mu_x * mu_y + SSIM_C1
    a2 = 2 * sxy + SSIM_C2
    b1 = mu_x ** 2 + mu_y ** 2 + SSIM_C1
    b2 = sxx + syy + SSIM_C2
    s_map = (a1 * a2) / (b1 * b2)
    n_valid = mask.sum()
    value = float((s_map * mask).sum() / (n_valid * 3))
    if not with_grad:
        return value
    m = mask / (n_valid * 3)
    ds_dmu = 2 * (mu_y * a2 * b1 - mu_x * a1 * a2) / (b1 * b1 * b2)
    ds_dsxx = -s_map / b2
    ds_dsxy = 2 * a1 / (b1 * b2)
    grad = (window_filter(m * (ds_dmu - 2 * mu_x * ds_dsxx - mu_y * ds_dsxy))
            + 2 * x * window_filter(m * ds_dsxx) + y * window_filter(m * ds_dsxy))
    return value, grad


def mse(a, b):
    """optimizer.py:114-118 (clipped sRGB)."""
    xa = np.clip(linear_to_srgb(np.clip(a, 0.0, None)), 0.0, 1.0)
    xb = np.clip(linear_to_srgb(np.clip(b, 0.0, None)), 0.0, 1.0)
    return float(np.mean((xa - xb) ** 2))


def psnr(a, b):
    """optimizer.py:121-125."""
    e = mse(a, b)
    return float("inf") if e == 0.0 else float(10.0 * np.log10(1.0 / e))


def loss(rendered, target, lam):
    """optimizer.py:128-152: (total, seed = d total / d linear render)."""
    xs, ys = linear_to_srgb(rendered), linear_to_srgb(target)
    diff = xs - ys
    l1 = float(np.mean(np.abs(diff)))
    d_l1 = np.sign(diff) / diff.size
    if lam > 0.0:
        s_val, d_s = ssim(xs, ys, with_grad=True)
        total = (1.0 - lam) * l1 + lam * (1.0 - s_val)
        d = (1.0 - lam) * d_l1 - lam * d_s
    else:
        total, d = l1, d_l1
    return total, d * dsrgb_dlinear(rendered)


def bounded_adam_step(params, grads, m, v, step, lr, lr_mult=1.0):
    """optimizer.py:173-204 on dicts of float64 arrays (in place); ``step``
    is the step count after increment.  Returns the non-finite count."""
    skips = 0
    for key in params:
        g = grads[key]
        bad = ~np.isfinite(g)
        skips += int(bad.sum())
        g = np.where(bad, 0.0, g)
        m[key] *= ADAM_BETA1
        m[key] += (1 - ADAM_BETA1) * g
        v[key] *= ADAM_BETA2
        v[key] += (1 - ADAM_BETA2) * g * g
        mh = m[key] / (1 - ADAM_BETA1 ** step)
        vh = v[key] / (1 - ADAM_BETA2 ** step)
        params[key] -= lr[key] * lr_mult * mh / (np.sqrt(vh) + ADAM_EPS)
    if "opacities" in params:
        np.clip(params["opacities"], OPACITY_MIN, ALPHA_MAX, out=params["opacities"])
    if "scales" in params:
        np.maximum(params["scales"], SCALE_MIN, out=params["scales"])
    if "quats" in params:
        q = params["quats"]
        q /= np.linalg.norm(q, axis=1, keepdims=True)
    return skips

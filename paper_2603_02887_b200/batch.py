"""Per-ray batched compositing on the device.

Mirrors the reference's per-ray API:

  composite_batch(model, alpha, emission, background, valid=None)
                                     compositor.py:84-171
  finite_diff_gradients(model, samples, background, eps=1e-5, seed=(1,1,1))
                                     adjoint.py:195-222
  SplatSample, SplatGradients        compositor.py:36-50, adjoint.py:64-73

backed by one fp64 scan kernel per ray (``csrc/batch.cu``, C-ABI
``nxs_composite_batch``).  numpy inputs give numpy outputs (the reference
semantics); float64 CUDA tensors stay on the device.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .camera import ALPHA_MAX
from .transmittance import VARIANT_IDS, as_model

__all__ = ["SplatSample", "SplatGradients", "composite_batch", "finite_diff_gradients"]

_OUT_KEYS = ("weights", "radiance", "residual", "k0", "overdraw", "e_k", "theta0", "t_k")


@dataclass(frozen=True)
class SplatSample:
    """One sorted per-ray contribution: depth, opacity, emitted radiance."""
    depth: float
    alpha: float
    emission: tuple

    def __post_init__(self) -> None:
        if not 0.0 <= self.alpha <= ALPHA_MAX:
            raise ValueError(f"alpha must be in [0, {ALPHA_MAX}], got {self.alpha}")
        if any(e < 0.0 for e in self.emission):
            raise ValueError(f"emission must be nonnegative, got {self.emission}")


@dataclass
class SplatGradients:
    """Per-splat gradients of a seeded scalar loss: ``d_alpha`` (seed-
    contracted) and ``d_emission`` (per channel)."""
    d_alpha: np.ndarray
    d_emission: np.ndarray


def _torch():
    import torch
    return torch


def composite_batch(model, alpha, emission, background, valid=None, stream=None) -> dict:
    """Composite R rays of N samples at once (fp64).  Returns ``weights``
    (R, N), ``radiance`` (R, 3), ``residual`` (R,), ``k0`` (R,) 0-based
    saturation index (N when none), ``overdraw`` (R,), ``e_k`` (R, 3),
    ``theta0`` (R, 3) and ``t_k`` (R,)."""
    torch = _torch()
    m = as_model(model)
    on_device = isinstance(alpha, torch.Tensor) and alpha.is_cuda
    a = torch.as_tensor(alpha, dtype=torch.float64)
    if a.ndim != 2:
        raise ValueError(f"alpha must be (R, N), got {tuple(a.shape)}")
    R, N = int(a.shape[0]), int(a.shape[1])
    e = torch.as_tensor(emission, dtype=torch.float64)
    if tuple(e.shape) != (R, N, 3):
        raise ValueError(f"emission must be (R, N, 3) = {(R, N, 3)}, got {tuple(e.shape)}")
    dev = torch.device("cuda")
    a = a.to(dev).contiguous()
    e = e.to(dev).contiguous()
    v = None
    if valid is not None:
        v = torch.as_tensor(valid).to(dev, dtype=torch.uint8).contiguous()
        if tuple(v.shape) != (R, N):
            raise ValueError(f"valid must be (R, N), got {tuple(v.shape)}")
    f64 = dict(dtype=torch.float64, device=dev)
    out = {"weights": torch.empty((R, N), **f64), "radiance": torch.empty((R, 3), **f64),
           "residual": torch.empty(R, **f64),
           "k0": torch.empty(R, dtype=torch.int64, device=dev),
           "overdraw": torch.empty(R, dtype=torch.int64, device=dev),
           "e_k": torch.empty((R, 3), **f64), "theta0": torch.empty((R, 3), **f64),
           "t_k": torch.empty(R, **f64)}
    bg = (ctypes.c_double * 3)(*[float(x) for x in np.asarray(background,
                                                             dtype=np.float64).reshape(3)])
    mod = _native.make_model(VARIANT_IDS[m.variant], m.param)
    _native._check(_native.lib().nxs_composite_batch(
        mod, a.data_ptr() if R * N else None, e.data_ptr() if R * N else None,
        None if v is None else v.data_ptr(), R, N, bg,
        *[out[k].data_ptr() if out[k].numel() else None for k in _OUT_KEYS],
        _native._stream_ptr(stream)))
    if on_device:
        return out
    return {k: t.cpu().numpy() for k, t in out.items()}


def _unpack(samples):
    """adjoint.py:76-80 (SplatSample-like objects)."""
    n = len(samples)
    alpha = np.array([s.alpha for s in samples], dtype=np.float64)
    emission = np.array([s.emission for s in samples], dtype=np.float64).reshape(n, 3)
    return n, alpha, emission


def finite_diff_gradients(model, samples, background, eps: float = 1e-5,
                          seed=(1.0, 1.0, 1.0)) -> SplatGradients:
    """Central differences of the forward composite: one batched launch of
    the 4n perturbed copies [alpha+, alpha-, emission+, emission-] of the
    ray (adjoint.py:195-222)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    seed = np.asarray(seed, dtype=np.float64)
    n, alpha, emission = _unpack(samples)
    if n == 0:
        return SplatGradients(np.zeros(0), np.zeros((0, 3)))
    rows = 4 * n
    alphas = np.tile(alpha, (rows, 1))
    emissions = np.tile(emission, (rows, 1, 1))
    r = np.arange(n)
    alphas[r, r] += eps
    alphas[n + r, r] -= eps
    emissions[2 * n + r, r, :] += eps
    emissions[3 * n + r, r, :] -= eps
    radiance = composite_batch(model, alphas, emissions, background)["radiance"]
    d_alpha_rgb = (radiance[:n] - radiance[n:2 * n]) / (2 * eps)
    d_em_diag = (radiance[2 * n:3 * n] - radiance[3 * n:]) / (2 * eps)
    return SplatGradients(d_alpha_rgb @ seed, d_em_diag * seed[None, :])

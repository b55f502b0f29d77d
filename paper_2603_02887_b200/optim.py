"""Train-step neighbours of the render path on the device (SURVEY §8 row
f2): the image loss with its adjoint seed and the bounded Adam step, so a
training step (render -> loss -> render_backward -> Adam) never leaves the
GPU.  Mirrors the reference ``nexsplat.optimizer`` names and semantics:

  loss(rendered, target, lam)       optimizer.py:128-152
  ssim(x, y, with_grad=False)       optimizer.py:75-111
  mse(a, b), psnr(a, b)             optimizer.py:114-125
  AdamState, bounded_adam_step      optimizer.py:157-204

Inputs may be numpy arrays (reference semantics: float results, numpy
seed/gradient, parameters updated in place) or CUDA tensors (device path:
results stay on the device, see :func:`loss_device`).  The kernels
(``csrc/train.cu``) compute the loss in fp64 from the fp32 device images;
Adam keeps fp32 moments next to the fp32 device parameters.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native

__all__ = [
    "SSIM_WINDOW", "SSIM_SIGMA", "SSIM_C1", "SSIM_C2",
    "ADAM_BETA1", "ADAM_BETA2", "ADAM_EPS", "PARAM_GROUPS",
    "ssim", "loss", "loss_device", "mse", "psnr", "AdamState", "bounded_adam_step",
]

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8
PARAM_GROUPS = ("centers", "scales", "quats", "opacities", "sh")

_ws_lock = threading.Lock()
_workspaces: dict = {}


def _torch():
    import torch
    return torch


def _is_tensor(x) -> bool:
    try:
        return isinstance(x, _torch().Tensor)
    except ImportError:  # pragma: no cover
        return False


def _dev_image(x):
    """(H, W, 3) image as a contiguous fp32 CUDA tensor."""
    torch = _torch()
    if _is_tensor(x):
        t = x.detach()
        if not t.is_cuda:
            t = t.cuda()
        return t.to(torch.float32).contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return torch.from_numpy(a).pin_memory().cuda(non_blocking=True)


def _workspace(h: int, w: int, device):
    torch = _torch()
    key = (device.index, h, w)
    with _ws_lock:
        ws = _workspaces.get(key)
        if ws is None:
            n = int(_native.lib().nxs_loss_workspace_bytes(h, w))
            ws = torch.empty(n, dtype=torch.uint8, device=device)
            _workspaces[key] = ws
    return ws


def _check_pair(x, y):
    if tuple(x.shape) != tuple(y.shape):
        raise ValueError(f"image shapes differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    if len(x.shape) != 3 or x.shape[2] != 3:
        raise ValueError(f"images must be (H, W, 3), got {tuple(x.shape)}")


def _run_loss(x, y, lam: float, flags: int, want_seed: bool, stream=None):
    torch = _torch()
    _check_pair(x, y)
    if not 0.0 <= lam <= 1.0:
        raise ValueError(f"ssim weight must be in [0, 1], got {lam}")
    h, w = int(x.shape[0]), int(x.shape[1])
    if lam > 0.0 and (h < SSIM_WINDOW or w < SSIM_WINDOW):
        raise ValueError(f"images must be at least {SSIM_WINDOW} pixels on each side")
    xd, yd = _dev_image(x), _dev_image(y)
    out = torch.empty(4, dtype=torch.float64, device=xd.device)
    seed = torch.empty_like(xd) if want_seed else None
    ws = _workspace(h, w, xd.device)
    _native._check(_native.lib().nxs_image_loss(
        xd.data_ptr(), yd.data_ptr(), h, w, float(lam), int(flags), out.data_ptr(),
        None if seed is None else seed.data_ptr(), ws.data_ptr(), _native._stream_ptr(stream)))
    return out, seed


def loss_device(rendered, target, lam: float, stream=None):
    """Device path of :func:`loss`: returns ``(stats, seed)`` with
    ``stats`` a float64 CUDA tensor (total, L1, SSIM, MSE) and ``seed`` the
    fp32 (H, W, 3) adjoint seed — no host synchronisation."""
    return _run_loss(rendered, target, float(lam), 0, True, stream)


def loss(rendered_linear, target_linear, lam: float):
    """(1 - lam) L1 + lam (1 - SSIM), both in sRGB; returns the scalar loss
    and the seed d loss / d linear render (numpy float64 for numpy inputs,
    the fp32 CUDA tensor for tensor inputs)."""
    out, seed = _run_loss(rendered_linear, target_linear, float(lam), 0, True)
    total = float(out[0].item())
    if _is_tensor(rendered_linear):
        return total, seed
    return total, seed.double().cpu().numpy()


def ssim(x, y, with_grad: bool = False):
    """Mean SSIM over fully-interior 11x11 windows of (H, W, 3) images; with
    ``with_grad`` also d(mean ssim)/dx."""
    out, seed = _run_loss(x, y, 1.0, _native.NXS_LOSS_SRGB_INPUT, with_grad)
    value = float(out[2].item())
    if not with_grad:
        return value
    grad = -seed  # total = 1 - SSIM at lam = 1
    return value, (grad if _is_tensor(x) else grad.double().cpu().numpy())


def mse(a_linear, b_linear) -> float:
    """Mean squared error between images, in clipped sRGB."""
    out, _ = _run_loss(a_linear, b_linear, 0.0, 0, False)
    return float(out[3].item())


def psnr(a_linear, b_linear) -> float:
    """10 log10(1 / MSE) on [0, 1] sRGB images; +inf for identical inputs."""
    err = mse(a_linear, b_linear)
    if err == 0.0:
        return float("inf")
    return float(10.0 * np.log10(1.0 / err))


@dataclass
class AdamState:
    """Adam moments (CUDA tensors: float32 for device parameters, float64
    for the numpy drop-in's float64 parameters) and counters; the
    non-finite gradient count lives on the device until read."""
    m: dict
    v: dict
    step: int = 0
    _skips: object = field(default=None, repr=False)

    @classmethod
    def for_params(cls, params: dict) -> "AdamState":
        torch = _torch()
        m, v = {}, {}
        for k, p in params.items():
            shape = tuple(p.shape)
            dt = torch.float32 if _is_tensor(p) else torch.float64
            m[k] = torch.zeros(shape, dtype=dt, device="cuda")
            v[k] = torch.zeros(shape, dtype=dt, device="cuda")
        return cls(m=m, v=v)

    @property
    def nan_skips(self) -> int:
        return 0 if self._skips is None else int(self._skips.item())


def bounded_adam_step(params: dict, grads: dict, state: AdamState, lr: dict,
                      lr_mult: float = 1.0, stream=None) -> None:
    """One Adam step followed by projection onto parameter bounds (opacities
    clamped to [1e-4, 1 - 1e-6], scales floored at 1e-6, quaternions
    renormalised); non-finite gradients are dropped and counted
    (reference optimizer.py:173-204).  CUDA tensor parameters (float32) are
    updated in place on the device; numpy parameters (the reference's
    float64 arrays) are updated in float64 on the device — no float32 round
    trip — and written back in place."""
    torch = _torch()
    unknown = set(params) - set(PARAM_GROUPS)
    if unknown:
        raise ValueError(f"unknown parameter groups {sorted(unknown)}")
    kinds = {_is_tensor(p) for p in params.values()}
    if len(kinds) > 1:
        raise ValueError("parameters must be all CUDA tensors or all numpy arrays")
    f64 = kinds == {False}
    dt = torch.float64 if f64 else torch.float32
    state.step += 1
    if state._skips is None:
        state._skips = torch.zeros(1, dtype=torch.int64, device="cuda")
    groups = (_native.AdamGroup * 5)()
    keep = []
    host = {}
    for i, key in enumerate(PARAM_GROUPS):
        if key not in params:
            continue
        p = params[key]
        if not f64:
            if not (p.is_cuda and p.dtype == torch.float32 and p.is_contiguous()):
                raise ValueError(f"{key}: device parameters must be contiguous fp32 CUDA tensors")
            pd = p
        else:
            pd = torch.as_tensor(np.ascontiguousarray(p, dtype=np.float64)).to("cuda")
            host[key] = (p, pd)
        g = grads[key]
        gd = (g.detach().to(device="cuda", dtype=dt).contiguous() if _is_tensor(g)
              else torch.as_tensor(np.ascontiguousarray(g, dtype=np.float64)).to(
                  device="cuda", dtype=dt))
        gd = gd.reshape(tuple(pd.shape))
        m, v = state.m[key], state.v[key]
        if tuple(m.shape) != tuple(pd.shape) or tuple(gd.shape) != tuple(pd.shape):
            raise ValueError(f"{key}: parameter, gradient and moment shapes differ")
        if m.dtype != dt:
            raise ValueError(f"{key}: Adam moments are {m.dtype}, parameters need {dt}")
        keep += [pd, gd]
        groups[i] = _native.AdamGroup(pd.data_ptr(), gd.data_ptr(), m.data_ptr(), v.data_ptr(),
                                      int(pd.numel()), float(lr[key]))
    step_fn = _native.lib().nxs_adam_step_f64 if f64 else _native.lib().nxs_adam_step
    _native._check(step_fn(groups, int(state.step), float(lr_mult), state._skips.data_ptr(),
                           _native._stream_ptr(stream)))
    for key, (p, pd) in host.items():
        p[...] = pd.cpu().numpy().reshape(np.shape(p))

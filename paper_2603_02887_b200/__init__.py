"""B200-native generalized-transmittance splat renderer (arXiv 2603.02887).

Drop-in for the reference package's image-renderer path (``nexsplat.render``:
``render``, ``render_forward_cached``, ``render_backward``,
``render_with_gradients``, ``SceneArrays``, ``RenderResult``) backed by the
hand-written sm_100a CUDA library ``lib/libnxs.so`` (C-ABI: include/nxs.h).
The host-side descriptors (``TransmittanceModel``, ``Camera``,
``GaussianPrimitive``) mirror the reference's so existing callers can switch
imports; the reference's own objects are accepted as well.  ``optim``
holds the device loss / SSIM / bounded Adam of the reference optimizer
(the train-step neighbours of the render path).
"""
from .camera import (
    ALPHA_EPS,
    ALPHA_MAX,
    DEFAULT_ALPHA_CUTOFF,
    NEAR_PLANE,
    SH_C0,
    SH_C1,
    Camera,
    GaussianPrimitive,
    quat_to_rot,
)
from .render import (
    DeviceScene,
    RenderResult,
    SceneArrays,
    backward_device,
    forward_backward_device,
    forward_device,
    render,
    render_backward,
    render_forward_cached,
    render_with_gradients,
    zero_grads_device,
)
from .transmittance import TransmittanceModel, model_from_config, model_to_config
from . import optim
from .optim import AdamState, bounded_adam_step, loss, mse, psnr, ssim

__version__ = "0.1.0"

__all__ = [
    "ALPHA_EPS", "ALPHA_MAX", "DEFAULT_ALPHA_CUTOFF", "NEAR_PLANE", "SH_C0", "SH_C1",
    "Camera", "GaussianPrimitive", "quat_to_rot",
    "DeviceScene", "RenderResult", "SceneArrays", "render", "render_forward_cached",
    "render_backward", "render_with_gradients", "forward_device", "backward_device",
    "forward_backward_device",
    "zero_grads_device",
    "TransmittanceModel", "model_from_config", "model_to_config",
    "optim", "AdamState", "bounded_adam_step", "loss", "mse", "psnr", "ssim",
]

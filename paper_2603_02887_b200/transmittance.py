"""Transmittance model descriptor (host side).

Mirrors the reference ``TransmittanceModel`` (reference
``pkg/src/nexsplat/transmittance.py:54-115``): a tagged variant plus one
shape parameter, validated once at construction.  The device kernels only
ever see ``(variant id, param)``; this module is the host-side config
object and the mapping onto the C-ABI ``nxs_model`` struct.

Any object with ``.variant`` and ``.param`` attributes (for example the
reference's own ``nexsplat.TransmittanceModel``) is accepted by the render
entry points, so callers can switch without touching their model objects.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

__all__ = [
    "TransmittanceModel",
    "model_from_config",
    "model_to_config",
    "VARIANT_IDS",
    "softplus_norm",
]

# reference transmittance.py:27-30
_POWER_LAW_V_EPS = 1e-4
_MIN_KAPPA = 10.0

# order is the C-ABI enum (include/nxs.h, NXS_MODEL_*)
VARIANT_IDS = {
    "exponential": 0,
    "linear": 1,
    "quadratic": 2,
    "blended": 3,
    "vicini": 4,
    "power_law": 5,
    "softplus": 6,
}

# reference transmittance.py:43-51
_PARAM_KEY = {
    "exponential": "",
    "linear": "",
    "quadratic": "c",
    "blended": "gamma",
    "vicini": "gamma",
    "power_law": "v",
    "softplus": "kappa",
}


@dataclass(frozen=True)
class TransmittanceModel:
    """Tagged transmittance variant plus its single shape parameter.

    Validation follows reference ``transmittance.py:66-79`` exactly so the
    same inputs raise the same ``ValueError``s.
    """

    variant: str
    param: float = 0.0

    def __post_init__(self) -> None:
        if self.variant not in VARIANT_IDS:
            raise ValueError(f"unknown transmittance variant: {self.variant!r}")
        p = self.param
        if not math.isfinite(p):
            raise ValueError(f"{self.variant}: parameter must be finite, got {p!r}")
        if self.variant == "quadratic" and p < -0.5:
            raise ValueError(f"quadratic curvature must be >= -0.5, got {p}")
        if self.variant in ("blended", "vicini") and not (0.0 <= p <= 1.0):
            raise ValueError(f"{self.variant} mix weight must be in [0, 1], got {p}")
        if self.variant == "power_law" and p < -1.0:
            raise ValueError(f"power-law exponent must be >= -1, got {p}")
        if self.variant == "softplus" and p < _MIN_KAPPA:
            raise ValueError(f"softplus sharpness must be >= {_MIN_KAPPA}, got {p}")

    @classmethod
    def exponential(cls) -> "TransmittanceModel":
        return cls("exponential")

    @classmethod
    def linear(cls) -> "TransmittanceModel":
        return cls("linear")

    @classmethod
    def quadratic(cls, c: float) -> "TransmittanceModel":
        return cls("quadratic", float(c))

    @classmethod
    def blended(cls, gamma: float) -> "TransmittanceModel":
        return cls("blended", float(gamma))

    @classmethod
    def vicini(cls, gamma: float) -> "TransmittanceModel":
        return cls("vicini", float(gamma))

    @classmethod
    def power_law(cls, v: float) -> "TransmittanceModel":
        return cls("power_law", float(v))

    @classmethod
    def softplus(cls, kappa: float) -> "TransmittanceModel":
        return cls("softplus", float(kappa))

    def describe(self) -> str:
        key = _PARAM_KEY[self.variant]
        if not key:
            return self.variant
        return f"{self.variant}({key}={self.param:g})"


def softplus_norm(kappa: float) -> float:
    """K = kappa / log(1 + e^kappa), the softplus weight normaliser
    (reference transmittance.py:262, ``k / _softplus_fn(k)``)."""
    # logaddexp(0, k) for k >= 10 without overflow
    return kappa / (kappa + math.log1p(math.exp(-kappa)))


def model_from_config(cfg: dict) -> TransmittanceModel:
    """reference transmittance.py:268-282."""
    if "model" not in cfg:
        raise ValueError("model config requires a 'model' tag")
    tag = str(cfg["model"]).lower().replace("-", "_")
    aliases = {"powerlaw": "power_law", "vicini_blend": "vicini", "exp": "exponential"}
    tag = aliases.get(tag, tag)
    if tag not in VARIANT_IDS:
        raise ValueError(f"unknown transmittance model tag: {cfg['model']!r}")
    key = _PARAM_KEY[tag]
    if not key:
        return TransmittanceModel(tag)
    if key not in cfg:
        raise ValueError(f"model {tag!r} requires parameter {key!r}")
    return TransmittanceModel(tag, float(cfg[key]))


def model_to_config(model) -> dict:
    cfg: dict = {"model": model.variant}
    key = _PARAM_KEY[model.variant]
    if key:
        cfg[key] = model.param
    return cfg


def as_model(model) -> TransmittanceModel:
    """Normalise any ``.variant/.param`` object (e.g. the reference's own
    model class) into this module's validated descriptor."""
    if isinstance(model, TransmittanceModel):
        return model
    try:
        return TransmittanceModel(str(model.variant), float(getattr(model, "param", 0.0)))
    except AttributeError as exc:  # pragma: no cover - defensive
        raise TypeError(f"not a transmittance model: {model!r}") from exc

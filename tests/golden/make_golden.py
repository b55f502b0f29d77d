"""Generate the golden fixtures by running the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Runs only in the build container (the reference is not on the GPU box);
the .npz files it writes are committed and are what the tests read.

Fixtures (all scenes are stored, so nothing is regenerated at test time):
  golden_small.npz    reference test scene (tests/test_primitives.py:243-248,
                      rng 31, 8 primitives, 24x16): forward outputs + cache for
                      7 models x chunk_size {None, 1}; render_backward
                      gradients for exp/linear/quadratic.
  golden_c1.npz       canonical scene at config C1 (1k Gaussians,
                      64x64, fp32-rounded), chunk_size=1: forward for 5 models,
                      render_backward for exp/linear/quadratic(0.5).
  golden_fd.npz       tiny scene (tests/test_primitives.py:337-343 pattern):
                      central finite differences of the reference forward for
                      softplus(20) and blended(0.5) (no reference analytic
                      backward exists for these, render.py:229-231).
  golden_transmit.npz transmittance-study overdraw totals (acceptance crit. 7,
                      tests/test_acceptance.py:210-225).
  golden_order.npz    _depth_chunks order of a 100k canonical scene, 2 views.
  golden_chunk.npz    chunked order (Mode C): the small scene at chunk_size 3
                      (7 models, + gradients for exp/linear/quadratic) and the
                      C1 scene at chunk_size 128 (the TrainConfig default,
                      reference optimizer.py:278) and 64, 5 models, gradients
                      for exp/linear/quadratic(0.5).
  golden_train.npz    train-step neighbours: loss() for lam 0 / 0.2 / 1 on
                      fp32-rounded 37x53 images (values over and below the
                      sRGB knee and above 1), ssim(x, y, with_grad=True),
                      mse/psnr, and three bounded_adam_step() calls on a
                      64-Gaussian parameter set (one gradient with NaN/inf).
  golden_batch.npz    composite_batch() of 300 rays x 40 samples (ragged
                      valid masks, saturating and non-saturating rays, an
                      exactly-saturating ray) for the 7 models, N = 0, and
                      finite_diff_gradients() of a 6-sample ray.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

from nexsplat.primitives import Camera, GaussianPrimitive  # noqa: E402
from nexsplat.render import (SceneArrays, _depth_chunks, render,  # noqa: E402
                             render_forward_cached, render_with_gradients)
from nexsplat.studies import transmit_study_camera, transmit_study_scene  # noqa: E402
from nexsplat.transmittance import TransmittanceModel as TM  # noqa: E402

from oracle import splat_oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent

MODELS = {
    "exponential": TM.exponential(),
    "linear": TM.linear(),
    "quadratic_0.5": TM.quadratic(0.5),
    "softplus_20": TM.softplus(20.0),
    "blended_0.5": TM.blended(0.5),
    "vicini_0.3": TM.vicini(0.3),
    "power_law_2": TM.power_law(2.0),
}
BWD = ("exponential", "linear", "quadratic_0.5")


def random_prim(rng, center_box=1.0, z=(2.0, 6.0)):
    """tests/test_primitives.py:36-42"""
    center = np.array([*rng.uniform(-center_box, center_box, 2), rng.uniform(*z)])
    scale = rng.uniform(0.2, 0.8, 3)
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    sh = rng.uniform(0.2, 2.0, (3, 4))
    return GaussianPrimitive(center, scale, q, rng.uniform(0.2, 0.9), sh)


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rounded(arrs):
    return SceneArrays(f32(arrs.centers), f32(arrs.scales), f32(arrs.quats),
                       f32(arrs.opacities), f32(arrs.sh))


def cam_dict(cam, prefix="cam_"):
    return {prefix + "position": cam.position, prefix + "rotation": cam.rotation,
            prefix + "focal": cam.focal, prefix + "cx": cam.cx, prefix + "cy": cam.cy,
            prefix + "width": cam.width, prefix + "height": cam.height}


def scene_dict(a, prefix="scene_"):
    return {prefix + k: getattr(a, k) for k in ("centers", "scales", "quats", "opacities", "sh")}


def small():
    rng = np.random.default_rng(31)
    scene = [random_prim(rng) for _ in range(8)]
    arrs = rounded(SceneArrays.from_primitives(scene))
    cam = Camera.from_look_at([0, 0, -3], [0, 0, 4], [0, 1, 0], 55.0, 24, 16)
    bg = f32([0.05, 0.1, 0.15])
    seed = f32(np.random.default_rng(7).uniform(0.2, 1.0, (16, 24, 3)))
    d = {**scene_dict(arrs), **cam_dict(cam), "bg": bg, "seed": seed}
    for name, m in MODELS.items():
        for cs in (None, 1):
            tag = f"{name}__{'none' if cs is None else cs}"
            res, cache = render_forward_cached(arrs, cam, m, bg, chunk_size=cs)
            d[tag + "__rgb"] = res.rgb
            d[tag + "__overdraw"] = res.overdraw
            d[tag + "__residual"] = res.residual
            for k in ("sat", "e_k", "t_k", "theta0"):
                d[tag + "__" + k] = cache[k]
            if name in BWD:
                _, g = render_with_gradients(arrs, cam, m, bg, seed, chunk_size=cs)
                for k, v in g.items():
                    d[tag + "__g_" + k] = v
    np.savez_compressed(OUT / "golden_small.npz", **d)


def c1():
    sc = O.round_scene_f32(O.canonical_scene(1000, seed=5))
    arrs = SceneArrays(sc.centers, sc.scales, sc.quats, sc.opacities, sc.sh)
    cam = Camera.from_look_at([0, 0, 0], [0, 0, 3.5], [0, 1, 0], 55.0, 64, 64)
    bg = f32([0.1, 0.05, 0.2])
    seed = f32(O.canonical_seed(64, 64, 0))
    d = {**scene_dict(arrs), **cam_dict(cam), "bg": bg, "seed": seed}
    for name in ("exponential", "linear", "quadratic_0.5", "softplus_20", "blended_0.5"):
        m = MODELS[name]
        if name in BWD:
            res, g = render_with_gradients(arrs, cam, m, bg, seed, chunk_size=1)
            for k, v in g.items():
                d[name + "__g_" + k] = v
        else:
            res = render(arrs, cam, m, bg, chunk_size=1)
        d[name + "__rgb"] = res.rgb
        d[name + "__overdraw"] = res.overdraw
        d[name + "__residual"] = res.residual
        print("c1", name, "mean overdraw", res.overdraw.mean())
    np.savez_compressed(OUT / "golden_c1.npz", **d)


def fd():
    rng = np.random.default_rng(41)
    scene = [random_prim(rng, center_box=0.6) for _ in range(4)]
    arrs = rounded(SceneArrays.from_primitives(scene))
    cam = Camera.from_look_at([0, 0, -3], [0, 0, 4], [0, 1, 0], 55.0, 12, 10)
    bg = f32([0.1, 0.05, 0.2])
    seed = f32(rng.uniform(0.2, 1.0, (10, 12, 3)))
    d = {**scene_dict(arrs), **cam_dict(cam), "bg": bg, "seed": seed}
    eps = 1e-6
    for name in ("softplus_20", "blended_0.5", "exponential", "linear"):
        m = MODELS[name]
        for cs in (None, 1):
            def scalar(a):
                return float(np.sum(seed * render(a, cam, m, bg, chunk_size=cs).rgb))
            out = {}
            for field in ("centers", "scales", "quats", "opacities", "sh"):
                base = getattr(arrs, field)
                g = np.zeros_like(base)
                for idx in np.ndindex(base.shape):
                    plus, minus = arrs.copy(), arrs.copy()
                    getattr(plus, field)[idx] += eps
                    getattr(minus, field)[idx] -= eps
                    g[idx] = (scalar(plus) - scalar(minus)) / (2 * eps)
                out[field] = g
            tag = f"{name}__{'none' if cs is None else cs}"
            for k, v in out.items():
                d[tag + "__fd_" + k] = v
    np.savez_compressed(OUT / "golden_fd.npz", **d)


def transmit():
    scene = transmit_study_scene(42)
    cam = transmit_study_camera(32)
    arrs = SceneArrays.from_primitives(scene)
    models = {"quadratic_1": TM.quadratic(1.0), "linear": TM.linear(),
              "quadratic_-0.5": TM.quadratic(-0.5), "exponential": TM.exponential(),
              "power_law_2": TM.power_law(2.0)}
    d = {**scene_dict(arrs), **cam_dict(cam)}
    for name, m in models.items():
        for cs in (None, 1):
            od = render(arrs, cam, m, np.zeros(3), chunk_size=cs).overdraw
            d[f"{name}__{'none' if cs is None else cs}__overdraw_total"] = int(od.sum())
            print("transmit", name, cs, int(od.sum()))
    np.savez_compressed(OUT / "golden_transmit.npz", **d)


def order():
    sc = O.round_scene_f32(O.canonical_scene(100_000, seed=5))
    arrs = SceneArrays(sc.centers, sc.scales, sc.quats, sc.opacities, sc.sh)
    d = {}  # the scene is regenerated by oracle.splat_oracle.canonical_scene(100_000, 5)
    for v in (0, 3):
        cam = Camera.from_look_at([0.4 * np.cos(2 * np.pi * v / 8), 0.4 * np.sin(2 * np.pi * v / 8),
                                   0.0], [0, 0, 3.5], [0, 1, 0], 55.0, 512, 512)
        chunks = _depth_chunks(arrs, cam, 1)
        d.update(cam_dict(cam, f"v{v}_cam_"))
        d[f"v{v}_order"] = np.concatenate(chunks).astype(np.int32)
    np.savez_compressed(OUT / "golden_order.npz", **d)


def chunk():
    d = {}
    rng = np.random.default_rng(31)
    scene = [random_prim(rng) for _ in range(8)]
    arrs = rounded(SceneArrays.from_primitives(scene))
    cam = Camera.from_look_at([0, 0, -3], [0, 0, 4], [0, 1, 0], 55.0, 24, 16)
    bg = f32([0.05, 0.1, 0.15])
    seed = f32(np.random.default_rng(7).uniform(0.2, 1.0, (16, 24, 3)))
    for name, m in MODELS.items():
        tag = f"small__{name}__3"
        res = render(arrs, cam, m, bg, chunk_size=3)
        d[tag + "__rgb"], d[tag + "__overdraw"], d[tag + "__residual"] = \
            res.rgb, res.overdraw, res.residual
        if name in BWD:
            _, g = render_with_gradients(arrs, cam, m, bg, seed, chunk_size=3)
            for k, v in g.items():
                d[tag + "__g_" + k] = v
    sc = O.round_scene_f32(O.canonical_scene(1000, seed=5))
    arrs = SceneArrays(sc.centers, sc.scales, sc.quats, sc.opacities, sc.sh)
    cam = Camera.from_look_at([0, 0, 0], [0, 0, 3.5], [0, 1, 0], 55.0, 64, 64)
    bg = f32([0.1, 0.05, 0.2])
    seed = f32(O.canonical_seed(64, 64, 0))
    for cs in (128, 64):
        for name in ("exponential", "linear", "quadratic_0.5", "softplus_20", "blended_0.5"):
            m = MODELS[name]
            tag = f"c1__{name}__{cs}"
            if name in BWD:
                res, g = render_with_gradients(arrs, cam, m, bg, seed, chunk_size=cs)
                for k, v in g.items():
                    d[tag + "__g_" + k] = v
            else:
                res = render(arrs, cam, m, bg, chunk_size=cs)
            d[tag + "__rgb"], d[tag + "__overdraw"], d[tag + "__residual"] = \
                res.rgb, res.overdraw, res.residual
            print("chunk", cs, name, "mean overdraw", res.overdraw.mean())
    np.savez_compressed(OUT / "golden_chunk.npz", **d)


def train():
    from nexsplat.optimizer import AdamState, bounded_adam_step, loss, mse, psnr, ssim
    rng = np.random.default_rng(17)
    H, W = 37, 53
    d = {}
    ren = f32(np.clip(rng.normal(0.4, 0.35, (H, W, 3)), -0.05, 1.3))
    ren[:3, :3] = 0.001  # below the sRGB knee
    tgt = f32(np.clip(ren + rng.normal(0, 0.1, (H, W, 3)), 0.0, 1.2))
    tgt[5, 5] = ren[5, 5]  # a zero difference (sign 0)
    d["rendered"], d["target"] = ren, tgt
    for lam in (0.0, 0.2, 1.0):
        total, seed = loss(ren, tgt, lam)
        d[f"loss_{lam}"] = total
        d[f"seed_{lam}"] = seed
    x, y = f32(rng.uniform(0, 1, (H, W, 3))), f32(rng.uniform(0, 1, (H, W, 3)))
    d["ssim_x"], d["ssim_y"] = x, y
    d["ssim_value"], d["ssim_grad"] = ssim(x, y, with_grad=True)
    d["mse"], d["psnr"] = mse(ren, tgt), psnr(ren, tgt)
    n = 64
    params = {"centers": f32(rng.normal(0, 1, (n, 3))),
              "scales": f32(rng.uniform(1e-6, 0.2, (n, 3))),
              "quats": f32(rng.normal(0, 1, (n, 4))),
              "opacities": f32(rng.uniform(0.0, 1.0, n)),
              "sh": f32(rng.normal(0, 0.5, (n, 3, 4)))}
    params["quats"] = f32(params["quats"] / np.linalg.norm(params["quats"], axis=1,
                                                          keepdims=True))
    for k, v in params.items():
        d["p0_" + k] = v.copy()
    state = AdamState.for_params(params)
    lr = {"centers": 0.13, "scales": 0.08, "quats": 0.45, "opacities": 1.0, "sh": 2.0}
    for step in range(3):
        grads = {k: f32(rng.normal(0, 0.3, v.shape)) for k, v in params.items()}
        if step == 1:
            grads["centers"][2, 1] = np.nan
            grads["sh"][5, 0, 0] = np.inf
        for k, v in grads.items():
            d[f"g{step}_{k}"] = v
        bounded_adam_step(params, grads, state, lr, lr_mult=0.9)
        for k, v in params.items():
            d[f"p{step + 1}_{k}"] = v.copy()
    d["nan_skips"] = state.nan_skips
    np.savez_compressed(OUT / "golden_train.npz", **d)


def batch():
    from nexsplat.adjoint import finite_diff_gradients
    from nexsplat.compositor import SplatSample, composite_batch
    rng = np.random.default_rng(23)
    R, N = 300, 40
    alpha = rng.uniform(0.0, 0.35, (R, N))
    alpha[:50] *= 0.1                      # rays that never saturate
    alpha[50:60, :3] = 0.999999            # early saturation
    alpha[60, :] = 0.0
    alpha[60, :4] = 0.25                   # linear: cumulative weight exactly 1 at i = 3
    emission = rng.uniform(0.0, 2.0, (R, N, 3))
    lengths = rng.integers(0, N + 1, R)
    valid = np.arange(N)[None, :] < lengths[:, None]
    valid[61] = rng.uniform(size=N) < 0.5  # holes inside a ray
    alpha = np.where(valid, alpha, 0.0)
    bg = np.array([0.1, 0.2, 0.3])
    d = {"alpha": alpha, "emission": emission, "valid": valid, "bg": bg}
    for name, m in MODELS.items():
        out = composite_batch(m, alpha, emission, bg, valid)
        for k, v in out.items():
            d[f"{name}__{k}"] = v
    out0 = composite_batch(MODELS["linear"], np.zeros((3, 0)), np.zeros((3, 0, 3)), bg)
    for k, v in out0.items():
        d[f"empty__{k}"] = v
    samples = [SplatSample(1.0 + i, float(a), tuple(float(x) for x in e))
               for i, (a, e) in enumerate(zip(rng.uniform(0.05, 0.5, 6),
                                              rng.uniform(0.1, 1.0, (6, 3))))]
    d["fd_alpha"] = np.array([s.alpha for s in samples])
    d["fd_emission"] = np.array([s.emission for s in samples])
    for name in ("exponential", "linear", "softplus_20", "blended_0.5"):
        g = finite_diff_gradients(MODELS[name], samples, bg, eps=1e-5, seed=(0.3, 1.0, 0.7))
        d[f"fd__{name}__d_alpha"] = g.d_alpha
        d[f"fd__{name}__d_emission"] = g.d_emission
    np.savez_compressed(OUT / "golden_batch.npz", **d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "c1", "fd", "transmit", "order", "chunk", "train", "batch"]
    for w in which:
        globals()[w]()
        print("wrote", w)

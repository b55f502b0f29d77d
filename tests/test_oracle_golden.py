"""Pin the CPU oracle to the reference: every golden vector produced by the
reference itself (tests/golden/make_golden.py) must be reproduced by
oracle/splat_oracle.py.  CPU only."""
import numpy as np
import pytest

from oracle import splat_oracle as O
from tests._util import GRAD_FIELDS, MODELS, cam_from, load, scene_from

SMALL = load("golden_small.npz")
C1 = load("golden_c1.npz")
FD = load("golden_fd.npz")


@pytest.mark.parametrize("cs", [None, 1])
@pytest.mark.parametrize("name", list(MODELS))
def test_forward_small_matches_reference(name, cs):
    d = SMALL
    tag = f"{name}__{'none' if cs is None else cs}"
    cam, sc, bg = cam_from(d), scene_from(d), d["bg"]
    out = O.forward(sc, cam, MODELS[name], bg, chunk_size=cs)
    H, W = cam.height, cam.width
    np.testing.assert_allclose(out["rad"].reshape(H, W, 3), d[tag + "__rgb"], atol=1e-12)
    np.testing.assert_array_equal(out["overdraw"].reshape(H, W), d[tag + "__overdraw"])
    np.testing.assert_allclose(out["residual"].reshape(H, W), d[tag + "__residual"], atol=1e-12)
    for k in ("e_k", "t_k", "theta0"):
        np.testing.assert_allclose(out[k], d[tag + "__" + k], atol=1e-12)
    np.testing.assert_array_equal(out["sat"], d[tag + "__sat"])


@pytest.mark.parametrize("cs", [None, 1])
@pytest.mark.parametrize("name", ["exponential", "linear", "quadratic_0.5"])
def test_backward_small_matches_reference(name, cs):
    d = SMALL
    tag = f"{name}__{'none' if cs is None else cs}"
    _, g = O.render_with_gradients(scene_from(d), cam_from(d), MODELS[name], d["bg"], d["seed"],
                                   chunk_size=cs)
    for k in GRAD_FIELDS:
        ref = d[tag + "__g_" + k]
        np.testing.assert_allclose(g[k], ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("name", ["exponential", "linear", "quadratic_0.5", "softplus_20",
                                  "blended_0.5"])
def test_c1_matches_reference(name):
    d = C1
    cam, sc = cam_from(d), scene_from(d)
    fwd, g = O.render_with_gradients(sc, cam, MODELS[name], d["bg"], d["seed"], chunk_size=1)
    H, W = cam.height, cam.width
    np.testing.assert_allclose(fwd["rad"].reshape(H, W, 3), d[name + "__rgb"], atol=1e-12)
    np.testing.assert_array_equal(fwd["overdraw"].reshape(H, W), d[name + "__overdraw"])
    if name + "__g_centers" in d:
        for k in GRAD_FIELDS:
            ref = d[name + "__g_" + k]
            np.testing.assert_allclose(g[k], ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("cs", [None, 1])
@pytest.mark.parametrize("name", ["softplus_20", "blended_0.5", "exponential", "linear"])
def test_backward_matches_reference_finite_differences(name, cs):
    """The unified adjoint vs central FD of the reference forward (the
    reference's only gradient oracle for softplus/blended); tolerance of
    reference tests/test_primitives.py:363 (rel 2e-4, abs 2e-6)."""
    d = FD
    tag = f"{name}__{'none' if cs is None else cs}"
    _, g = O.render_with_gradients(scene_from(d), cam_from(d), MODELS[name], d["bg"], d["seed"],
                                   chunk_size=cs)
    for k in GRAD_FIELDS:
        fd = d[tag + "__fd_" + k]
        np.testing.assert_allclose(g[k], fd, rtol=2e-4, atol=2e-6, err_msg=k)


def test_transmit_study_overdraw_totals():
    """Acceptance crit. 7 (reference tests/test_acceptance.py:210-225,
    pkg/test_output.txt:23)."""
    d = load("golden_transmit.npz")
    cam, sc = cam_from(d), scene_from(d)
    models = {"quadratic_1": ("quadratic", 1.0), "linear": ("linear", 0.0),
              "quadratic_-0.5": ("quadratic", -0.5), "exponential": ("exponential", 0.0),
              "power_law_2": ("power_law", 2.0)}
    expect = {"quadratic_1": 37888, "linear": 51200, "quadratic_-0.5": 93184,
              "exponential": 102400, "power_law_2": 102400}
    from tests._util import Model
    for name, (v, p) in models.items():
        for cs in (None, 1):
            out = O.forward(sc, cam, Model(v, p), np.zeros(3), chunk_size=cs)
            total = int(out["overdraw"].sum())
            assert total == int(d[f"{name}__{'none' if cs is None else cs}__overdraw_total"])
            assert total == expect[name]


def test_depth_order_matches_reference():
    d = load("golden_order.npz")
    sc = O.round_scene_f32(O.canonical_scene(100_000, seed=5))
    for v in (0, 3):
        cam = cam_from(d, f"v{v}_cam_")
        np.testing.assert_array_equal(O.depth_order(sc, cam), d[f"v{v}_order"])


def test_pixel_subset_is_exact():
    """Pixel batching reproduces the full image (SURVEY Probe P3)."""
    d = C1
    cam, sc = cam_from(d), scene_from(d)
    full = O.forward(sc, cam, MODELS["exponential"], d["bg"], chunk_size=1)
    px = np.random.default_rng(0).choice(cam.width * cam.height, 97, replace=False)
    sub = O.forward(sc, cam, MODELS["exponential"], d["bg"], chunk_size=1, pixels=px)
    np.testing.assert_array_equal(sub["rad"], full["rad"][px])
    np.testing.assert_array_equal(sub["overdraw"], full["overdraw"][px])


CHUNK = load("golden_chunk.npz")


@pytest.mark.parametrize("name", list(MODELS))
def test_chunked_small_matches_reference(name):
    """chunk_size=3 over the 8-primitive scene: per-pixel t order inside
    each chunk of 3 (reference render.py:350-358, 171)."""
    d, tag = SMALL, f"small__{name}__3"
    cam, sc, bg = cam_from(d), scene_from(d), d["bg"]
    H, W = cam.height, cam.width
    if tag + "__g_centers" in CHUNK:
        fwd, g = O.render_with_gradients(sc, cam, MODELS[name], bg, d["seed"], chunk_size=3)
        for k in GRAD_FIELDS:
            ref = CHUNK[tag + "__g_" + k]
            np.testing.assert_allclose(g[k], ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())
    else:
        fwd = O.forward(sc, cam, MODELS[name], bg, chunk_size=3)
    np.testing.assert_allclose(fwd["rad"].reshape(H, W, 3), CHUNK[tag + "__rgb"], atol=1e-12)
    np.testing.assert_array_equal(fwd["overdraw"].reshape(H, W), CHUNK[tag + "__overdraw"])
    np.testing.assert_allclose(fwd["residual"].reshape(H, W), CHUNK[tag + "__residual"],
                               atol=1e-12)


@pytest.mark.parametrize("cs", [128, 64])
@pytest.mark.parametrize("name", ["exponential", "linear", "quadratic_0.5", "softplus_20",
                                  "blended_0.5"])
def test_chunked_c1_matches_reference(name, cs):
    d, tag = C1, f"c1__{name}__{cs}"
    cam, sc = cam_from(d), scene_from(d)
    H, W = cam.height, cam.width
    fwd, g = O.render_with_gradients(sc, cam, MODELS[name], d["bg"], d["seed"], chunk_size=cs)
    np.testing.assert_allclose(fwd["rad"].reshape(H, W, 3), CHUNK[tag + "__rgb"], atol=1e-12)
    np.testing.assert_array_equal(fwd["overdraw"].reshape(H, W), CHUNK[tag + "__overdraw"])
    if tag + "__g_centers" in CHUNK:
        for k in GRAD_FIELDS:
            ref = CHUNK[tag + "__g_" + k]
            np.testing.assert_allclose(g[k], ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())


# ---------------------------------------------------------------------------
# train-step neighbours: oracle/train_oracle.py against
# the reference's loss / ssim / mse / psnr / bounded_adam_step
# ---------------------------------------------------------------------------
TRAIN = load("golden_train.npz")


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_train_oracle_loss_matches_reference(lam):
    from oracle import train_oracle as T
    total, seed = T.loss(TRAIN["rendered"], TRAIN["target"], lam)
    assert total == pytest.approx(float(TRAIN[f"loss_{lam}"]), rel=1e-13)
    np.testing.assert_allclose(seed, TRAIN[f"seed_{lam}"], rtol=1e-11,
                               atol=1e-14 * np.abs(TRAIN[f"seed_{lam}"]).max())


def test_train_oracle_ssim_mse_psnr_match_reference():
    from oracle import train_oracle as T
    v, g = T.ssim(TRAIN["ssim_x"], TRAIN["ssim_y"], with_grad=True)
    assert v == pytest.approx(float(TRAIN["ssim_value"]), rel=1e-13)
    np.testing.assert_allclose(g, TRAIN["ssim_grad"], rtol=1e-10,
                               atol=1e-14 * np.abs(TRAIN["ssim_grad"]).max())
    assert T.mse(TRAIN["rendered"], TRAIN["target"]) == pytest.approx(float(TRAIN["mse"]),
                                                                        rel=1e-13)
    assert T.psnr(TRAIN["rendered"], TRAIN["target"]) == pytest.approx(float(TRAIN["psnr"]),
                                                                         rel=1e-13)
    with pytest.raises(ValueError):
        T.ssim(np.zeros((10, 20, 3)), np.zeros((10, 20, 3)))


def test_train_oracle_adam_matches_reference():
    from oracle import train_oracle as T
    keys = ("centers", "scales", "quats", "opacities", "sh")
    params = {k: TRAIN["p0_" + k].copy() for k in keys}
    m = {k: np.zeros_like(v) for k, v in params.items()}
    v = {k: np.zeros_like(x) for k, x in params.items()}
    lr = {"centers": 0.13, "scales": 0.08, "quats": 0.45, "opacities": 1.0, "sh": 2.0}
    skips = 0
    for step in range(3):
        grads = {k: TRAIN[f"g{step}_{k}"] for k in keys}
        skips += T.bounded_adam_step(params, grads, m, v, step + 1, lr, 0.9)
        for k in keys:
            np.testing.assert_allclose(params[k], TRAIN[f"p{step + 1}_{k}"], rtol=1e-13,
                                       atol=1e-15)
    assert skips == int(TRAIN["nan_skips"]) == 2


# ---------------------------------------------------------------------------
# per-ray batched compositor: oracle/ray_oracle.py against
# the reference's composite_batch / finite_diff_gradients
# ---------------------------------------------------------------------------
BATCH = load("golden_batch.npz")
BATCH_KEYS = ("weights", "radiance", "residual", "k0", "overdraw", "e_k", "theta0", "t_k")


@pytest.mark.parametrize("name", list(MODELS))
def test_ray_oracle_composite_batch_matches_reference(name):
    from oracle import ray_oracle as RO
    m = MODELS[name]
    out = RO.composite_batch(m.variant, m.param, BATCH["alpha"], BATCH["emission"], BATCH["bg"],
                             BATCH["valid"])
    for k in BATCH_KEYS:
        np.testing.assert_allclose(out[k], BATCH[f"{name}__{k}"], rtol=1e-12, atol=1e-13,
                                   err_msg=k)


def test_ray_oracle_empty_and_finite_differences_match_reference():
    from oracle import ray_oracle as RO
    out = RO.composite_batch("linear", 0.0, np.zeros((3, 0)), np.zeros((3, 0, 3)), BATCH["bg"])
    for k in BATCH_KEYS:
        np.testing.assert_array_equal(out[k], BATCH[f"empty__{k}"], err_msg=k)
    for name in ("exponential", "linear", "softplus_20", "blended_0.5"):
        m = MODELS[name]
        da, de = RO.finite_diff_gradients(m.variant, m.param, BATCH["fd_alpha"],
                                          BATCH["fd_emission"], BATCH["bg"], 1e-5, (0.3, 1.0, 0.7))
        np.testing.assert_allclose(da, BATCH[f"fd__{name}__d_alpha"], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(de, BATCH[f"fd__{name}__d_emission"], rtol=1e-9, atol=1e-10)

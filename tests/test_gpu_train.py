"""GPU parity of the train-step neighbours: the device
loss / SSIM / MSE and the bounded Adam step (csrc/train.cu, through the
C-ABI) against the reference's own outputs (tests/golden/golden_train.npz)
and the pinned oracle (oracle/train_oracle.py).

Tolerances: the loss is computed in fp64 from the same fp32 inputs, so
scalars match to 1e-10 relative; the seed / gradient are returned in fp32
(rtol 1e-6); Adam runs in fp32 on fp32 parameters (rtol 1e-5 after three
steps)."""
import numpy as np
import pytest

from oracle import splat_oracle as O
from oracle import train_oracle as T
from tests._util import MODELS, load

pytestmark = pytest.mark.gpu
TRAIN = load("golden_train.npz")
KEYS = ("centers", "scales", "quats", "opacities", "sh")
LR = {"centers": 0.13, "scales": 0.08, "quats": 0.45, "opacities": 1.0, "sh": 2.0}


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_loss_matches_reference(lam):
    from paper_2603_02887_b200 import optim
    total, seed = optim.loss(TRAIN["rendered"], TRAIN["target"], lam)
    assert total == pytest.approx(float(TRAIN[f"loss_{lam}"]), rel=1e-10)
    ref = TRAIN[f"seed_{lam}"]
    np.testing.assert_allclose(seed, ref, rtol=1e-6, atol=1e-9 * np.abs(ref).max())


def test_ssim_mse_psnr_match_reference():
    from paper_2603_02887_b200 import optim
    v, g = optim.ssim(TRAIN["ssim_x"], TRAIN["ssim_y"], with_grad=True)
    assert v == pytest.approx(float(TRAIN["ssim_value"]), rel=1e-10)
    ref = TRAIN["ssim_grad"]
    np.testing.assert_allclose(g, ref, rtol=1e-6, atol=1e-9 * np.abs(ref).max())
    assert optim.ssim(TRAIN["ssim_x"], TRAIN["ssim_y"]) == pytest.approx(v, rel=1e-14)
    assert optim.mse(TRAIN["rendered"], TRAIN["target"]) == pytest.approx(float(TRAIN["mse"]),
                                                                            rel=1e-10)
    assert optim.psnr(TRAIN["rendered"], TRAIN["target"]) == pytest.approx(
        float(TRAIN["psnr"]), rel=1e-10)
    assert optim.psnr(TRAIN["target"], TRAIN["target"]) == float("inf")


def test_loss_1080p_matches_oracle_and_device_path():
    """Full-size image, device tensors in and out (no host round trip)."""
    import torch
    from paper_2603_02887_b200 import optim
    rng = np.random.default_rng(3)
    ren = rng.uniform(-0.02, 1.1, (1080, 1920, 3)).astype(np.float32)
    tgt = np.clip(ren + rng.normal(0, 0.05, ren.shape), 0, 1).astype(np.float32)
    stats, seed = optim.loss_device(torch.from_numpy(ren).cuda(), torch.from_numpy(tgt).cuda(),
                                    0.2)
    total, ref_seed = T.loss(ren.astype(np.float64), tgt.astype(np.float64), 0.2)
    assert float(stats[0]) == pytest.approx(total, rel=1e-10)
    np.testing.assert_allclose(seed.double().cpu().numpy(), ref_seed, rtol=1e-6,
                               atol=1e-9 * np.abs(ref_seed).max())


def test_bounded_adam_matches_reference():
    import torch
    from paper_2603_02887_b200 import optim
    params = {k: torch.from_numpy(TRAIN["p0_" + k].astype(np.float32)).cuda() for k in KEYS}
    state = optim.AdamState.for_params(params)
    for step in range(3):
        grads = {k: torch.from_numpy(TRAIN[f"g{step}_{k}"].astype(np.float32)).cuda()
                 for k in KEYS}
        optim.bounded_adam_step(params, grads, state, LR, lr_mult=0.9)
        for k in KEYS:
            np.testing.assert_allclose(params[k].double().cpu().numpy(),
                                       TRAIN[f"p{step + 1}_{k}"], rtol=1e-5, atol=1e-6, err_msg=k)
    assert state.nan_skips == int(TRAIN["nan_skips"]) == 2
    assert state.step == 3


def test_bounded_adam_numpy_params_in_place():
    """numpy (float64) parameters update in float64 on the device
    (nxs_adam_step_f64): the reference's own trajectory to ~1e-12, not to
    float32 precision."""
    from paper_2603_02887_b200 import optim
    params = {k: TRAIN["p0_" + k].copy() for k in KEYS}
    ids = {k: id(v) for k, v in params.items()}
    state = optim.AdamState.for_params(params)
    for step in range(3):
        grads = {k: TRAIN[f"g{step}_{k}"] for k in KEYS}
        optim.bounded_adam_step(params, grads, state, LR, lr_mult=0.9)
        for k in KEYS:
            assert id(params[k]) == ids[k] and params[k].dtype == np.float64
            np.testing.assert_allclose(params[k], TRAIN[f"p{step + 1}_{k}"], rtol=1e-11,
                                       atol=1e-13, err_msg=k)
    assert state.nan_skips == int(TRAIN["nan_skips"]) == 2


def test_device_training_steps_reduce_the_loss():
    """render -> loss -> render_backward -> Adam entirely on the device
    (the reference train() inner loop, optimizer.py:383-396)."""
    import torch
    from paper_2603_02887_b200 import DeviceScene, _native, backward_device, forward_device, optim
    from paper_2603_02887_b200.camera import Camera
    sc = O.round_scene_f32(O.canonical_scene(2000, seed=5))
    cam = Camera.from_look_at([0, 0, 0], [0, 0, 3.5], [0, 1, 0], 55.0, 96, 80)
    model = MODELS["exponential"]
    target_scene = DeviceScene.from_arrays(sc)
    view = _native.View()
    target, _, _ = forward_device(view, target_scene, cam, model, np.zeros(3), chunk_size=128)
    target = target.clone()
    # perturbed start
    rng = np.random.default_rng(0)
    start = O.Scene(sc.centers + rng.normal(0, 0.02, sc.centers.shape), sc.scales, sc.quats,
                    sc.opacities, sc.sh)
    dev = DeviceScene.from_arrays(start)
    params = {k: getattr(dev, k) for k in KEYS}
    state = optim.AdamState.for_params(params)
    losses = []
    for it in range(12):
        rgb, _, _ = forward_device(view, dev, cam, model, np.zeros(3), chunk_size=128)
        stats, seed = optim.loss_device(rgb, target, 0.2)
        grads = backward_device(view, dev, seed)
        optim.bounded_adam_step(params, grads, state, {k: 1e-3 for k in KEYS})
        losses.append(float(stats[0]))
    assert losses[-1] < 0.9 * losses[0], losses
    torch.cuda.synchronize()

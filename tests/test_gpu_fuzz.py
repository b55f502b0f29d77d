"""Randomised parity sweep: many small random scenes and cameras (varied
sizes, anisotropy, opacity, SH degree, camera pose and field of view,
Gaussians crossing the near plane) in every ordering mode and the four
north-star transmittances, forward and backward, against the pinned CPU
oracle under the SURVEY §8c protocol (tests/test_gpu_parity.py)."""
import numpy as np
import pytest

from oracle import splat_oracle as O
from tests._util import MODELS, check_grads, check_masked
from tests.test_gpu_parity import check_forward, gpu_run

pytestmark = pytest.mark.gpu

FUZZ_MODELS = ["exponential", "linear", "softplus_20", "blended_0.5"]


def random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(20, 400))
    C = int(rng.choice([1, 4]))
    centers = np.column_stack([rng.uniform(-1.5, 1.5, n), rng.uniform(-1.2, 1.2, n),
                               rng.uniform(0.3 if seed % 3 == 0 else 1.5, 7.0, n)])
    aniso = rng.uniform(0.2, 1.0, (n, 3)) ** (2 if seed % 2 else 1)
    scales = rng.uniform(0.03, 0.4, (n, 1)) * aniso
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opac = rng.uniform(0.05, 0.99, n)
    sh = np.zeros((n, 3, C))
    sh[:, :, 0] = rng.uniform(0.1, 1.2, (n, 3)) / O.SH_C0
    if C == 4:
        sh[:, :, 1:] = rng.normal(0.0, 0.3, (n, 3, 3))
    sc = O.round_scene_f32(O.Scene(centers, scales, quats, opac, sh))
    W, H = int(rng.integers(24, 72)), int(rng.integers(20, 60))
    pos = rng.normal(0, 0.3, 3) * [1, 1, 0.2]
    cam = O.look_at(pos, [rng.normal(0, 0.2), rng.normal(0, 0.2), 4.0], [0, 1, 0],
                    float(rng.uniform(35, 80)), W, H)
    bg = np.asarray(rng.uniform(0, 0.3, 3), dtype=np.float32).astype(np.float64)
    seed_img = np.asarray(rng.uniform(0.2, 1.0, (H, W, 3)), dtype=np.float32).astype(np.float64)
    return sc, cam, bg, seed_img


@pytest.mark.parametrize("cs", [1, 16, None])
@pytest.mark.parametrize("seed", range(12))
def test_random_scenes_match_oracle(seed, cs):
    sc, cam, bg, seed_img = random_case(seed)
    name = FUZZ_MODELS[seed % len(FUZZ_MODELS)]
    model = MODELS[name]
    fwd = O.forward(sc, cam, model, bg, chunk_size=cs, keep_state=True)
    keep = ~fwd["mask"]
    seed_m = seed_img.reshape(-1, 3) * keep[:, None]
    g_ref, mass = O.backward(sc, cam, model, bg, fwd, seed_m, with_mass=True)
    got = gpu_run(sc, cam, model, bg, seed=seed_m.reshape(cam.height, cam.width, 3),
                  chunk_size=cs)
    bad, kept = check_forward(got, fwd, fwd["mask"], cam.height, cam.width)
    assert bad == 0, (name, cs, bad, kept)
    check_masked(fwd, model, cs != 1, cam.width * cam.height)
    check_grads("fuzz", f"{seed}__{name}__{cs}", got["grads"], g_ref, mass)
    assert got["stats"]["n_overflow"] == 0

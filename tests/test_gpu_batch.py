"""GPU parity of the per-ray batched compositor (SURVEY §8 row f4,
csrc/batch.cu through the C-ABI) against the reference's own
composite_batch / finite_diff_gradients outputs
(tests/golden/golden_batch.npz) and the pinned oracle
(oracle/ray_oracle.py).  fp64 throughout: 1e-12 relative."""
import numpy as np
import pytest

from oracle import ray_oracle as RO
from tests._util import MODELS, load

pytestmark = pytest.mark.gpu
BATCH = load("golden_batch.npz")
KEYS = ("weights", "radiance", "residual", "k0", "overdraw", "e_k", "theta0", "t_k")


@pytest.mark.parametrize("name", list(MODELS))
def test_composite_batch_matches_reference(name):
    from paper_2603_02887_b200 import batch
    out = batch.composite_batch(MODELS[name], BATCH["alpha"], BATCH["emission"], BATCH["bg"],
                                BATCH["valid"])
    for k in KEYS:
        np.testing.assert_allclose(out[k], BATCH[f"{name}__{k}"], rtol=1e-12, atol=1e-13,
                                   err_msg=k)
    sat = BATCH[f"{name}__k0"] < BATCH["alpha"].shape[1]
    assert sat.any() and (~sat).any()  # both kinds of rays are covered


def test_composite_batch_empty_and_device_tensors():
    import torch
    from paper_2603_02887_b200 import batch
    out = batch.composite_batch(MODELS["linear"], np.zeros((3, 0)), np.zeros((3, 0, 3)),
                                BATCH["bg"])
    for k in KEYS:
        np.testing.assert_array_equal(out[k], BATCH[f"empty__{k}"], err_msg=k)
    a = torch.as_tensor(BATCH["alpha"]).cuda()
    e = torch.as_tensor(BATCH["emission"]).cuda()
    out = batch.composite_batch(MODELS["exponential"], a, e, BATCH["bg"], BATCH["valid"])
    assert out["radiance"].is_cuda
    np.testing.assert_allclose(out["radiance"].cpu().numpy(),
                               BATCH["exponential__radiance"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("name", ["exponential", "linear", "softplus_20", "blended_0.5"])
def test_finite_diff_gradients_match_reference(name):
    from paper_2603_02887_b200 import batch
    samples = [batch.SplatSample(1.0 + i, float(a), tuple(e))
               for i, (a, e) in enumerate(zip(BATCH["fd_alpha"], BATCH["fd_emission"]))]
    g = batch.finite_diff_gradients(MODELS[name], samples, BATCH["bg"], eps=1e-5,
                                    seed=(0.3, 1.0, 0.7))
    np.testing.assert_allclose(g.d_alpha, BATCH[f"fd__{name}__d_alpha"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(g.d_emission, BATCH[f"fd__{name}__d_emission"], rtol=1e-8,
                               atol=1e-10)


def test_composite_batch_large_matches_oracle():
    """100k rays x 128 samples (the render cap) against the oracle scan."""
    from paper_2603_02887_b200 import batch
    rng = np.random.default_rng(5)
    R, N = 100_000, 128
    alpha = rng.uniform(0, 0.08, (R, N))
    emission = rng.uniform(0, 1, (R, N, 3))
    m = MODELS["softplus_20"]
    out = batch.composite_batch(m, alpha, emission, np.zeros(3))
    ref = RO.composite_batch(m.variant, m.param, alpha[:2000], emission[:2000], np.zeros(3))
    for k in KEYS:
        np.testing.assert_allclose(out[k][:2000], ref[k], rtol=1e-12, atol=1e-13, err_msg=k)

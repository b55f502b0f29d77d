"""GPU parity at the north-star configuration C3 (BASELINE.json configs[1]:
1M Gaussians — the canonical scene, seed 5 — at 1920x1080), the workload the
bench headline is quoted on, through the steady-state path the bench times:
ONE reused ``nxs_view`` called several times, so the checked call runs the
device-sized first depth phase replayed as a CUDA graph and the fused
forward+backward with its speculative phase count.  Every transmittance
model in the global order (BASELINE north_star: "for every transmittance
function"), and the exact and chunked orders for three of them.

Sampled-pixel protocol: the oracle (``splat_oracle``, pruned
candidates — exact, see its module doc) evaluates N random pixels; the seed
is non-zero only on the unmasked samples, so every gradient entry of the 1M
scene is comparable.  Reference semantics: ``_forward_sweep`` /
``_backward_sweep`` (reference render.py:147-347) in the order of
``_depth_chunks`` (render.py:350-358) for chunk_size=1, per-pixel t order
(render.py:171) for chunk_size None / 128.

Asserted (BASELINE north_star tolerance, |x-ref| <= 1e-6 + 1e-5|ref|):
  * rgb and residual within tolerance, overdraw exact, on every unmasked
    sample;  samples masked for an alpha-cutoff / saturation decision margin
    <= 1 %.  The t-ordered modes also mask samples where two candidates' peak
    depths agree to 1e-6 relative: at 1M Gaussians that is
    ~1.6 % of Mode X pixels (measured, 4 of 256), so the total is capped at 3 %
    there (10 % for the exponential model, which composites 128 splats per
    pixel: 9 of 128), and the report counts how many masked samples matched
    anyway (all of them);
  * every gradient entry within the mass-scaled bound (normwise geometric
    scale), strict failures <= 0.1 % of the touched entries.
The componentwise-scale failure count is reported next to it.  Each case
writes its counts to ``$NXS_PARITY_DIR/c3`` (default gpurun_out/parity/c3/),
collected into profiles/r02_parity_c3.json.
"""
import numpy as np
import pytest

from oracle import splat_oracle as O
from tests._util import (GRAD_FIELDS, MODELS, check_grads, check_masked, close, mask_parts,
                         write_report)

pytestmark = pytest.mark.gpu

W, H, P = 1920, 1080, 1_000_000
CASES = [("exponential", 1, 256), ("linear", 1, 256), ("softplus_20", 1, 256),
         ("blended_0.5", 1, 256), ("quadratic_0.5", 1, 128), ("vicini_0.3", 1, 128),
         ("power_law_2", 1, 128), ("softplus_20", None, 256), ("softplus_20", 128, 256),
         ("exponential", None, 128), ("blended_0.5", 128, 128)]
CALLS = 3  # the checked call is the third on one view


@pytest.fixture(scope="module")
def c3():
    import torch
    from paper_2603_02887_b200 import DeviceScene
    sc = O.round_scene_f32(O.canonical_scene(P, seed=5))
    cam = O.canonical_camera(W, H)
    dev = DeviceScene.from_arrays(sc)
    seed_img = O.canonical_seed(W, H, 0).reshape(-1, 3).astype(np.float32).astype(np.float64)
    yield sc, cam, dev, seed_img
    del dev
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,cs,n_px", CASES,
                         ids=[f"{n}-{'none' if c is None else c}" for n, c, _ in CASES])
def test_c3_sampled_pixels_match_oracle(c3, name, cs, n_px):
    import torch
    from paper_2603_02887_b200 import _native, forward_backward_device
    sc, cam, dev, seed_img = c3
    model = MODELS[name]
    bg = np.zeros(3)
    px = np.random.default_rng(21 + (0 if cs == 1 else 1 if cs is None else 2)).choice(
        W * H, n_px, replace=False)  # (the same pixels for every model of an order)
    fwd = O.forward(sc, cam, model, bg, chunk_size=cs, pixels=px, keep_state=True, batch=8)
    keep = ~fwd["mask"]
    seed_px = seed_img[px] * keep[:, None]
    g_ref, mass = O.backward(sc, cam, model, bg, fwd, seed_px, with_mass=True)
    seed_full = np.zeros((W * H, 3), dtype=np.float32)
    seed_full[px] = seed_px
    seed = torch.as_tensor(seed_full.reshape(H, W, 3)).cuda()

    view = _native.View()
    launches = []
    for _ in range(CALLS):
        n0 = view.stats()["n_launches"]
        grads = {k: torch.zeros_like(getattr(dev, k)) for k in GRAD_FIELDS}
        out, grads = forward_backward_device(view, dev, cam, model, bg, seed, grads,
                                             chunk_size=cs)
        torch.cuda.synchronize()
        launches.append(view.stats()["n_launches"] - n0)
    rgb = out[0].double().cpu().numpy().reshape(-1, 3)[px]
    od = out[1].cpu().numpy().reshape(-1)[px]
    res = out[2].double().cpu().numpy().reshape(-1)[px]
    got = {k: v.double().cpu().numpy() for k, v in grads.items()}
    view.close()

    ok = close(rgb, fwd["rad"]).all(1) & (od == fwd["overdraw"]) & close(res, fwd["residual"])
    bad_px = int((keep & ~ok).sum())
    dec, tt = mask_parts(fwd, model, cs != 1)
    tag = f"{name}__{'none' if cs is None else cs}"
    extra = dict(case=name, chunk_size=cs, pixels=n_px, masked=int((~keep).sum()),
                 masked_decision=int(dec.sum()), masked_t_tie_only=int(tt.sum()),
                 masked_but_matching=int((~keep & ok).sum()), forward_failures=bad_px,
                 mean_overdraw=float(fwd["overdraw"].mean()), launches_per_call=launches)
    if bad_px:
        write_report("c3", tag, extra)
    assert bad_px == 0, extra
    check_grads("c3", tag, got, g_ref, mass, basis="touched", **extra)
    # t ties grow with the splats a pixel composites: the exponential model
    # never saturates and composites 128 (vs ~10), 9 of 128 Mode X pixels have
    # a pair within 1e-6 relative peak depth (all 9 matched anyway)
    check_masked(fwd, model, cs != 1, n_px,
                 t_cap=0.1 if model.variant == "exponential" else 0.03)

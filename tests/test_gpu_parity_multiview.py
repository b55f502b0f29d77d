"""GPU parity of the multi-view data-parallel step at the
BASELINE.json multi-view configurations, against the pinned CPU oracle:

  C4-like: the 1M-Gaussian scene at 1920x1080, softplus(20), 8 views of the
           canonical orbit (C4's per-rank share of 64 views over 8 GPUs);
  C5-like: the 5M-Gaussian scene at 3840x2160, blended(0.5), 2 views of
           C5's 256-view orbit.

Views run through ``device_view_renderer`` with FEWER workspaces than views
(each view's sizing history moves between workspaces) and
``DataParallelStep`` accumulating every view's gradients into one buffer;
the step runs twice, so the checked step clears the buffer through the
touched-row mask and reuses the histories.  Sampled pixels per view, seed
non-zero only there; the oracle sums the views' gradients.
Reference semantics: reference render.py:147-347, 350-358 per view, summed
as the reference optimizer would over views (optimizer.py:393-408).
"""
import numpy as np
import pytest

from oracle import splat_oracle as O
from tests._util import (GRAD_FIELDS, MODELS, check_grads, check_masked, close, write_report)

pytestmark = pytest.mark.gpu

CASES = {
    "c4_8views": dict(P=1_000_000, W=1920, H=1080, model="softplus_20", views=list(range(8)),
                      orbit=8, pool=3, px=48),
    "c5_2views": dict(P=5_000_000, W=3840, H=2160, model="blended_0.5", views=[0, 128],
                      orbit=256, pool=1, px=48),
}


@pytest.mark.parametrize("case", list(CASES))
def test_multiview_dp_step_matches_oracle(case):
    import torch
    from paper_2603_02887_b200 import DeviceScene
    from paper_2603_02887_b200.dp import DataParallelStep, GradBuffer, device_view_renderer
    c = CASES[case]
    P, W, H, model = c["P"], c["W"], c["H"], MODELS[c["model"]]
    sc = O.round_scene_f32(O.canonical_scene(P, seed=5))
    cams = {v: O.canonical_camera(W, H, v, c["orbit"]) for v in c["views"]}
    rng = np.random.default_rng(41)
    g_ref = None
    mass = None
    seeds, pix, fwds = {}, {}, {}
    for v in c["views"]:
        px = rng.choice(W * H, c["px"], replace=False)
        fwd = O.forward(sc, cams[v], model, np.zeros(3), chunk_size=1, pixels=px,
                        keep_state=True, batch=8)
        keep = ~fwd["mask"]
        s = rng.uniform(0.2, 1.0, (len(px), 3)).astype(np.float32).astype(np.float64)
        s *= keep[:, None]
        g, m = O.backward(sc, cams[v], model, np.zeros(3), fwd, s, with_mass=True)
        if g_ref is None:
            g_ref, mass = g, m
        else:
            for k in g_ref:
                g_ref[k] += g[k]
            for k in mass:
                mass[k] += m[k]
        img = np.zeros((W * H, 3), np.float32)
        img[px] = s
        seeds[v] = torch.as_tensor(img.reshape(H, W, 3)).cuda()
        pix[v], fwds[v] = px, fwd
    dev = DeviceScene.from_arrays(sc)
    order = list(c["views"])
    cam_list = [cams[v] for v in order]
    seed_list = [seeds[v] for v in order]
    inner = device_view_renderer(dev, model, np.zeros(3), cam_list, seed_list, pool=c["pool"])
    got_px = {}

    def render_view(i, grads):  # keep each view's sampled outputs before the slot is reused
        inner(i, grads)
        rgb, od, res = inner.outputs[i % c["pool"]]
        v = order[i]
        idx = torch.as_tensor(pix[v], device="cuda")
        got_px[v] = (rgb.reshape(-1, 3)[idx].double().cpu().numpy(),
                     od.reshape(-1)[idx].cpu().numpy(), res.reshape(-1)[idx].double().cpu().numpy())

    grads = GradBuffer(P, 4, device="cuda")
    step = DataParallelStep(len(order), 0, 1, grads, render_view)
    for _ in range(2):
        g = step()
        torch.cuda.synchronize()
    stats = [w.stats() for w in inner.workspaces]
    got = {k: v.double().cpu().numpy() for k, v in g.fields.items()}
    bad_px = 0
    for v in order:
        fwd = fwds[v]
        rgb, od, res = got_px[v]
        ok = close(rgb, fwd["rad"]).all(1) & (od == fwd["overdraw"]) & close(res, fwd["residual"])
        bad_px += int((~fwd["mask"] & ~ok).sum())
        check_masked(fwd, model, False, len(pix[v]))
    extra = dict(case=case, views=order, pool=c["pool"], pixels_per_view=c["px"],
                 forward_failures=bad_px, redone=sum(s["n_redo"] for s in stats))
    if bad_px:
        write_report("multiview", case, extra)
    assert bad_px == 0, extra
    check_grads("multiview", case, got, g_ref, mass, basis="touched", **extra)
    assert set(GRAD_FIELDS) == set(got)

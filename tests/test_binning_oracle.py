"""The C restatement of projection + binning (the bit-exact checker for the
device) against the reference semantics: its depth order is the
reference's _depth_chunks order, and its tile sets contain every
(Gaussian, pixel) pair the reference deems valid.  CPU only."""
import numpy as np
import pytest

import oracle
from oracle import splat_oracle as O
from tests._util import assert_order_matches_up_to_ties, cam_from, exact_depths, load


def test_order_matches_reference_golden():
    """Same order as the reference's _depth_chunks except between
    Gaussians whose depths agree to <= 4 ulps."""
    d = load("golden_order.npz")
    sc = O.round_scene_f32(O.canonical_scene(100_000, seed=5))
    for v in (0, 3):
        cam = cam_from(d, f"v{v}_cam_")
        b = oracle.binning(sc, cam)
        n = assert_order_matches_up_to_ties(b["order"], d[f"v{v}_order"],
                                            exact_depths(sc.centers, cam))
        assert n <= 10


def test_order_is_sorted_by_exact_depth():
    sc = O.round_scene_f32(O.canonical_scene(20_000, seed=9))
    cam = O.canonical_camera(64, 64, 5, 8)
    b = oracle.binning(sc, cam)
    dep = exact_depths(sc.centers, cam)[b["order"]].astype(np.float64)
    assert (np.diff(dep) >= 0).all()


@pytest.mark.parametrize("n,W,H,view", [(300, 64, 48, 0), (5000, 160, 120, 3)])
def test_tile_sets_cover_reference_valid_pairs(n, W, H, view):
    sc = O.round_scene_f32(O.canonical_scene(n, seed=view))
    cam = O.canonical_camera(W, H, view, 8)
    b = oracle.binning(sc, cam)
    rank = np.empty(n, int)
    rank[b["order"]] = np.arange(n)
    dirs = O.pixel_directions(cam)
    for s0 in range(0, n, 1000):
        ids = np.arange(s0, min(n, s0 + 1000))
        g = O._geometry(sc, ids, dirs, cam.position, 1e-4, 1 / 255)
        r_, m_ = np.nonzero(g["valid"])
        rc = b["rects"][rank[ids[r_]]]
        tx, ty = (m_ % W) // 16, (m_ // W) // 16
        assert ((rc[:, 0] <= tx) & (tx <= rc[:, 2]) & (rc[:, 1] <= ty) & (ty <= rc[:, 3])).all()


def test_pair_lists_are_rank_ordered_per_tile():
    sc = O.round_scene_f32(O.canonical_scene(2000, seed=1))
    cam = O.canonical_camera(128, 96)
    b = oracle.binning(sc, cam)
    for t0, t1 in b["ranges"]:
        seg = b["pairs"][t0:t1]
        assert (np.diff(seg) > 0).all()
    assert b["ranges"][:, 1].max() == b["n_pairs"]


def test_record_conic_reproduces_reference_alpha():
    """fp32 evaluation of the record vs reference fp64 α:
    all within 1e-6 + 1e-5|α| and identical validity."""
    f32 = np.float32
    n, W, H = 4000, 128, 96
    sc = O.round_scene_f32(O.canonical_scene(n, seed=5))
    cam = O.canonical_camera(W, H)
    b = oracle.binning(sc, cam)
    rank = np.empty(n, int)
    rank[b["order"]] = np.arange(n)
    ids = np.arange(n)
    g = O._geometry(sc, ids, O.pixel_directions(cam), cam.position, 1e-4, 1 / 255)
    r = b["records"][rank[ids]]
    j, i = np.arange(W * H) % W, np.arange(W * H) // W
    pxc, pyc = (j + 0.5).astype(f32), (i + 0.5).astype(f32)
    hx = ((j + 0.5 - cam.cx) / cam.focal).astype(f32)
    hy = ((i + 0.5 - cam.cy) / cam.focal).astype(f32)
    R = lambda k: r[:, k][:, None]  # noqa: E731
    ddx, ddy = (pxc[None] - R(0)) - R(2), (pyc[None] - R(1)) - R(3)
    w = R(5) * ddy + ddx
    num = (R(4) * w) * w + (R(6) * ddy) * ddy
    u, v = (R(9) * hy[None] + R(10)) + hx[None], hy[None] + R(12)
    D = (R(8) * u) * u + ((R(11) * v) * v + R(13))
    alpha = np.minimum(R(14) * np.exp(f32(-0.5) * (num / D)), f32(0.999999))
    valid = (num <= R(7) * D) & (alpha >= f32(1 / 255))
    assert (valid == g["valid"]).all()
    a, ref = alpha[valid], g["alpha"][valid]
    assert (np.abs(a - ref) <= 1e-6 + 1e-5 * ref).all()

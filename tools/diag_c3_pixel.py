"""Diagnostic: every gradient field of one Gaussian from ONE pixel's seed,
GPU vs oracle, in the three ordering modes (C3 scene).
usage: python tools/diag_c3_pixel.py MODEL GID PIXEL"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from oracle import splat_oracle as O  # noqa: E402
from paper_2603_02887_b200 import DeviceScene, _native, forward_backward_device  # noqa: E402
from tests._util import GRAD_FIELDS, MODELS  # noqa: E402

name, gid, p = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
W, H = 1920, 1080
sc = O.round_scene_f32(O.canonical_scene(1_000_000, seed=5))
cam = O.canonical_camera(W, H)
dev = DeviceScene.from_arrays(sc)
model = MODELS[name]
bg = np.zeros(3)
seed = O.canonical_seed(W, H, 0).reshape(-1, 3)[p:p + 1].astype(np.float32).astype(np.float64)
for cs in (1, None, 128):
    fwd = O.forward(sc, cam, model, bg, chunk_size=cs, pixels=np.array([p]), keep_state=True)
    g_ref = O.backward(sc, cam, model, bg, fwd, seed)
    s = np.zeros((W * H, 3), np.float32)
    s[p] = seed[0]
    st = torch.as_tensor(s.reshape(H, W, 3)).cuda()
    view = _native.View()
    g = {k: torch.zeros_like(getattr(dev, k)) for k in GRAD_FIELDS}
    out, g = forward_backward_device(view, dev, cam, model, bg, st, g, chunk_size=cs)
    torch.cuda.synchronize()
    print(f"== chunk {cs}: rgb gpu {out[0].reshape(-1, 3)[p].tolist()} ref {fwd['rad'][0]} "
          f"od {int(out[1].reshape(-1)[p])}/{fwd['overdraw'][0]} tmargin {fwd['tmargin'][0]:.3e}")
    st0 = fwd["_states"][0][3]
    order = st0["order"][:, 0]
    ids = st0["ids"]
    tt = st0["geo"]["t"][order, 0]
    vv = st0["geo"]["valid"][order, 0]
    aa = st0["geo"]["alpha"][order, 0]
    for i in range(min(int(fwd["overdraw"][0]) + 1, len(order))):
        if vv[i]:
            print(f"   slot {i}: gid {ids[order[i]]} t {tt[i]:.9f} alpha {aa[i]:.6f}")
    for k in GRAD_FIELDS:
        a = g[k][gid].double().cpu().numpy().ravel()
        b = g_ref[k][gid].ravel()
        print(f"  {k}: gpu {np.array2string(a, precision=9)}\n  {' ' * len(k)}  ref "
              f"{np.array2string(b, precision=9)}\n  {' ' * len(k)}  rel "
              f"{np.array2string((a - b) / (np.abs(b) + 1e-30), precision=2)}")
    view.close()

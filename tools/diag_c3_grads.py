"""Diagnostic: C3 sampled-pixel gradient failures, attributed per pixel.

For each failing gradient entry of a C3 case (tests/test_gpu_parity_c3.py),
re-render with the seed on ONE sampled pixel at a time (GPU and oracle) and
report the pixels whose contribution to that entry disagrees, with the
pixel's oracle t-order around the Gaussian.
usage: python tools/diag_c3_grads.py MODEL CHUNK(1|none|128)"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from oracle import splat_oracle as O  # noqa: E402
from paper_2603_02887_b200 import DeviceScene, _native, forward_backward_device  # noqa: E402
from tests._util import ATOL, GRAD_FIELDS, MODELS, RTOL  # noqa: E402

name = sys.argv[1]
cs = None if sys.argv[2] == "none" else int(sys.argv[2])
W, H = 1920, 1080
sc = O.round_scene_f32(O.canonical_scene(1_000_000, seed=5))
cam = O.canonical_camera(W, H)
dev = DeviceScene.from_arrays(sc)
model = MODELS[name]
bg = np.zeros(3)
px = np.random.default_rng(21 + (0 if cs == 1 else 1 if cs is None else 2)).choice(
    W * H, 256, replace=False)
seed_img = O.canonical_seed(W, H, 0).reshape(-1, 3).astype(np.float32).astype(np.float64)
fwd = O.forward(sc, cam, model, bg, chunk_size=cs, pixels=px, keep_state=True, batch=8)
keep = ~fwd["mask"]
seed_px = seed_img[px] * keep[:, None]
g_ref, mass = O.backward(sc, cam, model, bg, fwd, seed_px, with_mass=True)
view = _native.View()


def gpu(seed_rows, pixels):
    s = np.zeros((W * H, 3), np.float32)
    s[pixels] = seed_rows
    st = torch.as_tensor(s.reshape(H, W, 3)).cuda()
    g = {k: torch.zeros_like(getattr(dev, k)) for k in GRAD_FIELDS}
    for _ in range(2):
        for k in g:
            g[k].zero_()
        forward_backward_device(view, dev, cam, model, bg, st, g, chunk_size=cs)
    torch.cuda.synchronize()
    return {k: v.double().cpu().numpy() for k, v in g.items()}


got = gpu(seed_px, px)
report = []
for k in ("centers", "scales", "quats", "opacities", "sh"):
    err = np.abs(got[k] - g_ref[k])
    bad = np.argwhere(err > ATOL + RTOL * mass[k + "_c" if k + "_c" in mass else k])
    for b in bad:
        gid = int(b[0])
        ent = {"field": k, "index": b.tolist(), "got": float(got[k][tuple(b)]),
               "ref": float(g_ref[k][tuple(b)]), "mass": float(mass[k][tuple(b)]), "pixels": []}
        for b_px, idx, out, st in fwd["_states"]:
            if gid not in set(st["ids"].tolist()):
                continue
            for j, i in enumerate(idx):
                if not keep[i]:
                    continue
                gr = O._zero_grads(O.Scene.of(sc))
                one = np.zeros((len(idx), 3))
                one[j] = seed_px[i]
                O._backward_batch(O.Scene.of(sc), cam, model, bg, out, st, one, gr, None)
                if gr[k][tuple(b)] == 0:
                    continue
                gg = gpu(seed_px[i:i + 1], [px[i]])
                ent["pixels"].append({"pixel": int(px[i]), "got": float(gg[k][tuple(b)]),
                                      "ref": float(gr[k][tuple(b)]),
                                      "tmargin": float(fwd["tmargin"][i]),
                                      "overdraw": int(fwd["overdraw"][i])})
        report.append(ent)
        print(json.dumps(ent), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/diag_c3_{name}_{sys.argv[2]}.json").write_text(json.dumps(report, indent=1))

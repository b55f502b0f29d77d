"""Diagnostic: dump GPU vs oracle gradients (with mass) at C1 for analysis."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import splat_oracle as O
from tests._util import MODELS, cam_from, load, scene_from
from tests.test_gpu_parity import gpu_run

d = load("golden_c1.npz")
cam, sc, bg = cam_from(d), scene_from(d), d["bg"]
out = {}
for name in ["exponential", "linear", "softplus_20", "blended_0.5", "quadratic_0.5"]:
    model = MODELS[name]
    fwd = O.forward(sc, cam, model, bg, chunk_size=1, keep_state=True)
    seed = d["seed"].reshape(-1, 3) * (~fwd["mask"])[:, None]
    g_ref, mass = O.backward(sc, cam, model, bg, fwd, seed, with_mass=True)
    got = gpu_run(sc, cam, model, bg, seed=seed.reshape(cam.height, cam.width, 3))
    for k in g_ref:
        out[f"{name}__{k}__gpu"] = got["grads"][k]
        out[f"{name}__{k}__ref"] = g_ref[k]
        out[f"{name}__{k}__mass"] = mass[k]
    out[f"{name}__mask"] = fwd["mask"]
    out[f"{name}__rgb_gpu"] = got["rgb"]
    out[f"{name}__rgb_ref"] = fwd["rad"]
np.savez_compressed("gpurun_out/diag_grads.npz", **out)
print("ok")

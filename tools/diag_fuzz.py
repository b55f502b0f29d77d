"""Diagnostic: one fuzz case (tests/test_gpu_fuzz.py) — print the gradient
entries that fail the mass-scaled bound, with their Gaussian's geometry."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import splat_oracle as O
from tests._util import ATOL, GRAD_FIELDS, MODELS, RTOL
from tests.test_gpu_fuzz import FUZZ_MODELS, random_case
from tests.test_gpu_parity import gpu_run

seed = int(sys.argv[1]); cs = None if sys.argv[2] == "none" else int(sys.argv[2])
name = sys.argv[3] if len(sys.argv) > 3 else FUZZ_MODELS[seed % len(FUZZ_MODELS)]
sc, cam, bg, seed_img = random_case(seed)
model = MODELS[name]
fwd = O.forward(sc, cam, model, bg, chunk_size=cs, keep_state=True)
keep = ~fwd["mask"]
seed_m = seed_img.reshape(-1, 3) * keep[:, None]
g_ref, mass = O.backward(sc, cam, model, bg, fwd, seed_m, with_mass=True)
got = gpu_run(sc, cam, model, bg, seed=seed_m.reshape(cam.height, cam.width, 3), chunk_size=cs)
st = got["stats"]
print("n", len(sc.opacities), "W,H", cam.width, cam.height, "straddling", st["n_straddling"],
      "masked px", int((~keep).sum()))
bad_g = set()
for k in GRAD_FIELDS:
    a, b, m = got["grads"][k], g_ref[k], mass[k]
    bad = np.abs(a - b) > ATOL + RTOL * m
    for idx in zip(*np.nonzero(bad)):
        g = idx[0]
        bad_g.add(g)
        print(k, idx, "gpu %.6e ref %.6e mass %.3e diff %.3e" % (a[idx], b[idx], m[idx], a[idx] - b[idx]))
for g in sorted(bad_g):
    c = sc.centers[g]
    d = (c - cam.position) @ np.asarray(cam.rotation)[:, 2]
    print("g", g, "depth %.4f" % d, "scales", np.round(sc.scales[g], 4), "opac %.3f" % sc.opacities[g])

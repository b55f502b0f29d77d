"""Diagnostic: the strict-bound failures of one fuzz case (err vs |ref| vs
the componentwise mass), to tell cancellation-limited sums from errors.
usage: python tools/diag_fuzz_strict.py SEED CHUNK"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import splat_oracle as O  # noqa: E402
from tests._util import GRAD_FIELDS, MODELS, close  # noqa: E402
from tests.test_gpu_fuzz import FUZZ_MODELS, random_case  # noqa: E402
from tests.test_gpu_parity import gpu_run  # noqa: E402

seed = int(sys.argv[1])
cs = None if sys.argv[2] == "none" else int(sys.argv[2])
sc, cam, bg, seed_img = random_case(seed)
model = MODELS[FUZZ_MODELS[seed % len(FUZZ_MODELS)]]
fwd = O.forward(sc, cam, model, bg, chunk_size=cs, keep_state=True)
keep = ~fwd["mask"]
seed_m = seed_img.reshape(-1, 3) * keep[:, None]
g_ref, mass = O.backward(sc, cam, model, bg, fwd, seed_m, with_mass=True)
got = gpu_run(sc, cam, model, bg, seed=seed_m.reshape(cam.height, cam.width, 3), chunk_size=cs)
for k in GRAD_FIELDS:
    a, b = got["grads"][k], g_ref[k]
    m = mass.get(k + "_c", mass[k])
    for ix in np.argwhere(~close(a, b)):
        ix = tuple(ix)
        err = abs(a[ix] - b[ix])
        print(f"{k}{list(ix)} got {a[ix]:+.9e} ref {b[ix]:+.9e} err {err:.3e} "
              f"strict_tol {1e-6 + 1e-5 * abs(b[ix]):.3e} mass_c {m[ix]:.3e} "
              f"err/mass_tol {err / (1e-6 + 1e-5 * m[ix]):.3f} |ref|/mass {abs(b[ix]) / m[ix]:.2e}")

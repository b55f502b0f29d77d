"""Extended randomised parity sweep (beyond tests/test_gpu_fuzz.py):
python tools/fuzz_sweep.py START COUNT — every model, every ordering mode."""
import sys, traceback
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import splat_oracle as O
from tests._util import MODELS, grad_report
from tests.test_gpu_fuzz import random_case
from tests.test_gpu_parity import check_forward, gpu_run

start, count = int(sys.argv[1]), int(sys.argv[2])
names = list(MODELS)
fails = 0
for seed in range(start, start + count):
    sc, cam, bg, seed_img = random_case(seed)
    name = names[seed % len(names)]
    for cs in (1, 16, None):
        try:
            model = MODELS[name]
            fwd = O.forward(sc, cam, model, bg, chunk_size=cs, keep_state=True)
            keep = ~fwd["mask"]
            seed_m = seed_img.reshape(-1, 3) * keep[:, None]
            g_ref, mass = O.backward(sc, cam, model, bg, fwd, seed_m, with_mass=True)
            got = gpu_run(sc, cam, model, bg, seed=seed_m.reshape(cam.height, cam.width, 3),
                          chunk_size=cs)
            bad, kept = check_forward(got, fwd, fwd["mask"], cam.height, cam.width)
            strict, massf, total = grad_report(got["grads"], g_ref, mass)
            ok = bad == 0 and massf == 0 and kept >= 0.8 * cam.width * cam.height
            if not ok:
                fails += 1
                print(f"FAIL seed {seed} {name} cs={cs}: bad px {bad} kept {kept} "
                      f"strict {strict} mass {massf}/{total}")
        except Exception as e:
            fails += 1
            print(f"ERROR seed {seed} {name} cs={cs}: {e}")
print(f"done {count} seeds, {fails} failures")

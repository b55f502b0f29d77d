"""Per-pixel gradient comparison for one Gaussian of a fuzz case: seed one
pixel at a time and compare the GPU gradient with the oracle's."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import splat_oracle as O
from tests._util import MODELS
from tests.test_gpu_fuzz import FUZZ_MODELS, random_case
from tests.test_gpu_parity import gpu_run

seed, cs, gid, field, comp = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
sc, cam, bg, seed_img = random_case(seed)
model = MODELS[FUZZ_MODELS[seed % len(FUZZ_MODELS)]]
fwd = O.forward(sc, cam, model, bg, chunk_size=cs, keep_state=True)
W, H = cam.width, cam.height
full = seed_img.reshape(-1, 3)
rows = []
for p in range(W * H):
    s = np.zeros((W * H, 3)); s[p] = full[p]
    g_ref, mass = O.backward(sc, cam, model, bg, fwd, s, with_mass=True)
    r = g_ref[field][gid][comp] if g_ref[field].ndim == 2 else g_ref[field][gid]
    if r == 0.0:
        continue
    got = gpu_run(sc, cam, model, bg, seed=s.reshape(H, W, 3), chunk_size=cs)
    v = got["grads"][field][gid][comp]
    rows.append((abs(v - r) / (abs(r) + 1e-30), p, v, r, fwd["overdraw"][p], fwd["sat"][p]))
rows.sort(reverse=True)
for rel, p, v, r, od, sat in rows[:12]:
    print(f"px {p} (x={p % W}, y={p // W}) rel {rel:.2e} gpu {v:.6e} ref {r:.6e} overdraw {od} sat {sat}")
print("pixels", len(rows), "sum ref", sum(x[3] for x in rows), "sum gpu", sum(x[2] for x in rows))

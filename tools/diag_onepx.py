"""All gradient components of one Gaussian for a single seeded pixel."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import splat_oracle as O
from tests._util import MODELS, GRAD_FIELDS
from tests.test_gpu_fuzz import FUZZ_MODELS, random_case
from tests.test_gpu_parity import gpu_run

seed, cs, gid, p = (int(x) for x in sys.argv[1:5])
sc, cam, bg, seed_img = random_case(seed)
model = MODELS[FUZZ_MODELS[seed % len(FUZZ_MODELS)]]
fwd = O.forward(sc, cam, model, bg, chunk_size=cs, keep_state=True)
W, H = cam.width, cam.height
s = np.zeros((W * H, 3)); s[p] = seed_img.reshape(-1, 3)[p]
g_ref, mass = O.backward(sc, cam, model, bg, fwd, s, with_mass=True)
got = gpu_run(sc, cam, model, bg, seed=s.reshape(H, W, 3), chunk_size=cs)
for k in GRAD_FIELDS:
    print(k, "gpu", np.array2string(got["grads"][k][gid].ravel(), precision=7),
          "\n   ref", np.array2string(g_ref[k][gid].ravel(), precision=7))
print("cam pos", cam.position, "rot\n", np.asarray(cam.rotation), "focal", cam.focal)
print("center", sc.centers[gid], "scales", sc.scales[gid], "quat", sc.quats[gid])

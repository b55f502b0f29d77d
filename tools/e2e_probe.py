"""Break down the host-API (numpy) render_with_gradients time at C3."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import importlib  # noqa: E402
R = importlib.import_module("paper_2603_02887_b200.render")
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed  # noqa
from paper_2603_02887_b200.transmittance import TransmittanceModel  # noqa: E402

arrs = canonical_scene(1_000_000, seed=5)
arrs = R.SceneArrays(arrs.centers.astype(np.float64), arrs.scales.astype(np.float64),
                     arrs.quats.astype(np.float64), arrs.opacities.astype(np.float64),
                     arrs.sh.astype(np.float64))
cam = canonical_camera(1920, 1080)
seed = canonical_seed(1920, 1080, 0)
model = TransmittanceModel.softplus(20.0)


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    t0 = tick()
    dev = R.DeviceScene.from_arrays(arrs)
    t1 = tick()
    view = R._acquire_view()
    out = R.forward_device(view, dev, cam, model, np.zeros(3), chunk_size=1)
    t2 = tick()
    seed_t = R._h2d_f32(seed, dev.centers.device, "seed")
    t3 = tick()
    g = R.backward_device(view, dev, seed_t)
    t4 = tick()
    res = R._result_to_host(out)
    t5 = tick()
    dl = R._Download()
    for k, v in g.items():
        dl.add(v, "g_" + k)
    gh = dl.result()
    t6 = tick()
    R._release_view(view)
    t7 = time.perf_counter()
    R.render_with_gradients(arrs, cam, model, np.zeros(3), seed, chunk_size=1)
    t8 = tick()
    print(f"upload {1e3*(t1-t0):.2f} fwd {1e3*(t2-t1):.2f} seed {1e3*(t3-t2):.2f} "
          f"bwd {1e3*(t4-t3):.2f} fwd_d2h {1e3*(t5-t4):.2f} grads_d2h {1e3*(t6-t5):.2f} "
          f"| whole call {1e3*(t8-t7):.2f} ms")

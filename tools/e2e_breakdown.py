"""Where the numpy drop-in's time goes at C3 (render_with_gradients):
host->device upload of the scene and seed, the fused device call, the
downloads.  usage: python tools/e2e_breakdown.py"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_02887_b200 as nx  # noqa: E402
import importlib  # noqa: E402
R = importlib.import_module("paper_2603_02887_b200.render")
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed  # noqa

arrs = canonical_scene(1_000_000, seed=5)
cam = canonical_camera(1920, 1080)
seed = canonical_seed(1920, 1080)
m = nx.TransmittanceModel.softplus(20.0)
print("torch threads", torch.get_num_threads())
for _ in range(3):
    nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=1)
torch.cuda.synchronize()


def t(f, n=5):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


up = t(lambda: R.DeviceScene.from_arrays(arrs))
sd = t(lambda: R._h2d_f32(seed, torch.device("cuda"), "seed"))
dev = R.DeviceScene.from_arrays(arrs)
st = R._h2d_f32(seed, torch.device("cuda"), "seed")
view = R._acquire_view()
fb = t(lambda: R.forward_backward_device(view, dev, cam, m, np.zeros(3), st, chunk_size=1))
out, g = R.forward_backward_device(view, dev, cam, m, np.zeros(3), st, chunk_size=1)


def down():
    dl = R._Download()
    for x in list(out) + list(g.values()):
        dl.add(x)
    dl.result()


dn = t(down)
full = t(lambda: nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=1))
print(f"scene upload {up:.2f} ms, seed upload {sd:.2f} ms, fused device call {fb:.2f} ms, "
      f"downloads {dn:.2f} ms, sum {up + sd + fb + dn:.2f} ms; whole call {full:.2f} ms")
x = torch.empty(1 << 25, dtype=torch.float32, pin_memory=True)
y = torch.empty(1 << 25, dtype=torch.float32, device="cuda")
h2d = t(lambda: y.copy_(x, non_blocking=True))
d2h = t(lambda: x.copy_(y, non_blocking=True))
print(f"pinned DMA of 128 MiB: H2D {128 / 1.048576 / h2d:.1f} GB/s, D2H {128 / 1.048576 / d2h:.1f} GB/s")
a64 = np.random.rand(1 << 24)
cv = t(lambda: torch.from_numpy(a64).to(torch.float32))
print(f"host fp64->fp32 of 128 MiB fp64: {cv:.2f} ms")

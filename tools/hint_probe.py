"""Per-call behaviour of repeated fused calls on persistent views: wall time
(synchronised), depth phases and pair count.  Shows the first-phase hint
settling (global order) for the bench's multi-view cameras and for the
numpy API path."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_02887_b200 import (DeviceScene, _native, forward_backward_device,  # noqa: E402
                                   render_with_gradients)
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed  # noqa
from paper_2603_02887_b200.transmittance import TransmittanceModel  # noqa: E402

n_views = int(sys.argv[1]) if len(sys.argv) > 1 else 8
arrs = canonical_scene(1_000_000, seed=5)
dev = DeviceScene.from_arrays(arrs)
model = TransmittanceModel.softplus(20.0)
cams = [canonical_camera(1920, 1080, v, n_views) for v in range(n_views)]
seeds = [torch.as_tensor(canonical_seed(1920, 1080, v), dtype=torch.float32, device="cuda")
         for v in range(n_views)]
views = [_native.View().set_timing(True) for _ in range(n_views)]
for rep in range(5):
    line = []
    for v in range(n_views):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        forward_backward_device(views[v], dev, cams[v], model, np.zeros(3), seeds[v])
        torch.cuda.synchronize()
        st = views[v].stats()
        tm = views[v].timings()
        line.append(f"{1e3 * (time.perf_counter() - t0):.2f}ms/{int(tm['n_depth_phases'])}ph/"
                    f"{st['n_pairs'] // 1000}k")
    print("rep", rep, " ".join(line), flush=True)

cam = canonical_camera(1920, 1080)
seed = canonical_seed(1920, 1080, 0)
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    render_with_gradients(arrs, cam, model, np.zeros(3), seed, chunk_size=1)
    torch.cuda.synchronize()
    print(f"e2e call {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)

"""e2e A/B: render_with_gradients at C3 with the dense gradient download
(NXS_DENSE_GRADS=1) vs touched rows + background zero fill; plus host
zero-fill timings.  usage: python tools/e2e_probe2.py"""
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
for n, f in (("np.zeros+touch", lambda: np.zeros((1_000_000, 23)).__setitem__(
        (slice(None, None, 33),), 1.0)), ("torch.zeros", lambda: torch.zeros(1_000_000, 23,
                                                                             dtype=torch.float64))):
    f()
    t = time.perf_counter()
    for _ in range(5):
        f()
    print(n, (time.perf_counter() - t) / 5 * 1e3, "ms", flush=True)
if len(sys.argv) == 1:
    for dense in ("1", "0"):
        env = dict(os.environ, NXS_DENSE_GRADS=dense)
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True,
                             text=True)
        print("dense" if dense == "1" else "touched", out.stdout.strip()[-300:], out.stderr[-500:])
else:
    import paper_2603_02887_b200 as nx
    from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed
    arrs = canonical_scene(1_000_000, seed=5)
    cam = canonical_camera(1920, 1080)
    seed = canonical_seed(1920, 1080)
    m = nx.TransmittanceModel.softplus(20.0)
    for _ in range(3):
        r, g = nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=1)
    ts = []
    for _ in range(8):
        t = time.perf_counter()
        r, g = nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=1)
        ts.append(time.perf_counter() - t)
    print("ms", [round(x * 1e3, 2) for x in ts], "median", round(np.median(ts) * 1e3, 2),
          "Mpix/s", round(1920 * 1080 / np.median(ts) / 1e6, 1))

"""Device timeline of the bench step (C3, Mode G by default) from the CUDA
activity trace (torch.profiler / CUPTI): every kernel and copy of a few
steady-state steps with its start offset, duration and the idle gap before
it, and the host time per step.  Not a timing source for bench numbers.

    python tools/timeline_probe.py [chunk]   (chunk: 1 | 128 | none)
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_02887_b200 import DeviceScene  # noqa: E402
from paper_2603_02887_b200.dp import DataParallelStep, GradBuffer, device_view_renderer  # noqa
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed  # noqa
from paper_2603_02887_b200.transmittance import TransmittanceModel  # noqa: E402

chunk = sys.argv[1] if len(sys.argv) > 1 else "1"
chunk = None if chunk == "none" else int(chunk)
arrs = canonical_scene(1_000_000, seed=5)
dev = DeviceScene.from_arrays(arrs)
cams = [canonical_camera(1920, 1080)]
seeds = {0: torch.as_tensor(canonical_seed(1920, 1080, 0), dtype=torch.float32, device="cuda")}
grads = GradBuffer(len(arrs), arrs.sh.shape[2], device="cuda")
rv = device_view_renderer(dev, TransmittanceModel.softplus(20.0), np.zeros(3), cams, seeds,
                          chunk_size=chunk)
step = DataParallelStep(1, 0, 1, grads, rv)
for _ in range(10):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3 * (t1 - t0) / 20:.3f} ms/step, wall {1e3 * (t2 - t0) / 20:.3f} ms/step")

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(4):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
# print the last two steps
start_names = [i for i, e in enumerate(evs) if "k_depth" in e.name]
lo = start_names[-2] if len(start_names) >= 2 else 0
prev_end = None
t_first = evs[lo].time_range.start
busy = 0.0
for e in evs[lo:]:
    st, en = e.time_range.start, e.time_range.end
    gap = (st - prev_end) if prev_end is not None else 0.0
    busy += en - st
    print(f"{st - t_first:9.1f} us  +{gap:6.1f} gap  {en - st:7.1f} us  {e.name[:80]}")
    prev_end = max(prev_end or en, en)
span = prev_end - t_first
print(f"two steps: span {span:.1f} us, kernels/copies busy {busy:.1f} us")

"""Time the per-ray batched compositor (csrc/batch.cu) on device-resident
inputs: R rays x N samples, fp64, CUDA events after warm-up.  Reports rays/s
and achieved HBM bandwidth against the algorithmic 41 B per sample (alpha 8,
emission 24, weight 8, valid 1).  The reference's numpy composite_batch
(oracle port) is timed beside it on a bounded sample.

    python tools/bench_batch.py [--rays 1000000] [--samples 128]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2603_02887_b200 import batch  # noqa: E402
from paper_2603_02887_b200.transmittance import TransmittanceModel  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rays", type=int, default=1_000_000)
    p.add_argument("--samples", type=int, default=128)
    p.add_argument("--reps", type=int, default=10)
    a = p.parse_args()
    R, N = a.rays, a.samples
    g = torch.Generator(device="cuda").manual_seed(0)
    alpha = torch.rand(R, N, device="cuda", dtype=torch.float64, generator=g) * 0.05
    emission = torch.rand(R, N, 3, device="cuda", dtype=torch.float64, generator=g)
    valid = torch.ones(R, N, device="cuda", dtype=torch.uint8)
    model = TransmittanceModel.softplus(20.0)
    for _ in range(3):
        batch.composite_batch(model, alpha, emission, np.zeros(3), valid)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(a.reps):
        batch.composite_batch(model, alpha, emission, np.zeros(3), valid)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.reps
    nbytes = R * N * 41
    # reference-style numpy port on a bounded sample (oracle = test infrastructure)
    from oracle import ray_oracle as RO
    r_cpu = 20_000
    al, em = alpha[:r_cpu].cpu().numpy(), emission[:r_cpu].cpu().numpy()
    t0 = time.perf_counter()
    RO.composite_batch("softplus", 20.0, al, em, np.zeros(3))
    cpu_s = time.perf_counter() - t0
    print(json.dumps({"rays": R, "samples": N, "ms": round(ms, 4),
                      "rays_per_s": round(R / ms * 1e3), "GBps": round(nbytes / ms / 1e6, 1),
                      "cpu_port_rays_per_s": round(r_cpu / cpu_s),
                      "note": "with the 6 small per-ray outputs; includes the Python launch"}))


if __name__ == "__main__":
    main()

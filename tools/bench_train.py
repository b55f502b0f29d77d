"""Time the train-step neighbours at C3 (1M Gaussians, 1920x1080): the
device loss (L1 + SSIM + seed), the bounded Adam step, and a whole device
training step (forward -> loss -> backward -> Adam).  CUDA-event timing on
the current stream after warm-up; prints one JSON line.

    python tools/bench_train.py [--chunk 128] [--model exponential]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2603_02887_b200 import (DeviceScene, _native, backward_device,  # noqa: E402
                                   forward_device, optim, zero_grads_device)
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene  # noqa: E402
from paper_2603_02887_b200.transmittance import TransmittanceModel  # noqa: E402


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gaussians", type=int, default=1_000_000)
    p.add_argument("--chunk", default="128")
    p.add_argument("--model", default="exponential")
    p.add_argument("--reps", type=int, default=20)
    a = p.parse_args()
    chunk = None if a.chunk.lower() == "none" else int(a.chunk)
    W, H = 1920, 1080
    model = TransmittanceModel(a.model, {"softplus": 20.0, "blended": 0.5,
                                         "quadratic": 0.5}.get(a.model, 0.0))
    dev = DeviceScene.from_arrays(canonical_scene(a.gaussians, seed=5))
    cam = canonical_camera(W, H)
    view = _native.View()
    bg = np.zeros(3)
    target = torch.rand(H, W, 3, device="cuda")
    rgb, _, _ = forward_device(view, dev, cam, model, bg, chunk_size=chunk)
    KEYS = optim.PARAM_GROUPS
    params = {k: getattr(dev, k) for k in KEYS}
    state = optim.AdamState.for_params(params)
    grads = zero_grads_device(dev)
    lr = {k: 1e-6 for k in KEYS}
    for _ in range(3):
        optim.loss_device(rgb, target, 0.2)
        optim.bounded_adam_step(params, grads, state, lr)
    t_loss = timed(lambda: optim.loss_device(rgb, target, 0.2), a.reps)
    t_adam = timed(lambda: optim.bounded_adam_step(params, grads, state, lr), a.reps)

    def step():
        out, _, _ = forward_device(view, dev, cam, model, bg, chunk_size=chunk)
        _, seed = optim.loss_device(out, target, 0.2)
        g = backward_device(view, dev, seed)
        optim.bounded_adam_step(params, g, state, lr)
    for _ in range(3):
        step()
    t_step = timed(step, max(3, a.reps // 2))
    npix = W * H
    # algorithmic HBM bytes: loss reads 2 images (fp32), writes/reads 3 fp64
    # gradient maps and writes the fp32 seed; Adam reads p,g,m,v and writes p,m,v
    loss_bytes = npix * 3 * (4 + 4) * 2 + npix * 3 * 8 * 3 * 2 + npix * 3 * 4
    n_param = sum(t.numel() for t in params.values())
    adam_bytes = n_param * 4 * 7
    print(json.dumps({
        "workload": f"{a.gaussians} Gaussians, {W}x{H}, {model.describe()}, chunk_size={chunk}",
        "loss_ms": round(t_loss, 4), "loss_GBps": round(loss_bytes / t_loss / 1e6, 1),
        "adam_ms": round(t_adam, 4), "adam_GBps": round(adam_bytes / t_adam / 1e6, 1),
        "train_step_ms": round(t_step, 4),
        "train_step_mpix_s": round(npix / t_step / 1e3, 1)}))


if __name__ == "__main__":
    main()

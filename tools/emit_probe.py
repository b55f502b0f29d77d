"""Tile-emission workload at C3 (global order, warm view): how many ranks
the first depth phase emits, their candidate tile counts (rect areas) and
the lane efficiency of k_emit_tiles' warp-per-rank schedule.
Usage (GPU): python tools/emit_probe.py"""
import importlib

import numpy as np
import torch

from oracle import splat_oracle as O
from paper_2603_02887_b200 import DeviceScene, TransmittanceModel, _native

render = importlib.import_module("paper_2603_02887_b200.render")


def main():
    P, W, H = 1_000_000, 1920, 1080
    sc = O.round_scene_f32(O.canonical_scene(P, seed=5))
    cam = O.canonical_camera(W, H, 0, 8)
    dev = DeviceScene.from_arrays(sc)
    seed = torch.as_tensor(O.canonical_seed(W, H, 0), dtype=torch.float32).cuda()
    view = _native.View()
    grads = {k: torch.zeros_like(getattr(dev, k)) for k in ("centers", "scales", "quats", "opacities", "sh")}
    model = TransmittanceModel.softplus(20.0)
    for _ in range(3):
        render.forward_backward_device(view, dev, cam, model, np.zeros(3), seed, grads, chunk_size=1)
    torch.cuda.synchronize()
    T = ((W + 15) // 16) * ((H + 15) // 16)
    rects = torch.full((P, 4), -7, dtype=torch.int32, device="cuda")
    ranges = torch.zeros((T, 2), dtype=torch.int32, device="cuda")
    pairs = torch.full((8_000_000,), -7, dtype=torch.int32, device="cuda")
    view.binning_export(rects, ranges, pairs)
    order = torch.zeros(P, dtype=torch.int32, device="cuda")
    view.depth_order(order)
    torch.cuda.synchronize()
    r, p = ranges.cpu().numpy(), pairs.cpu().numpy()
    n = int(r[-1, 1])
    ranks = p[:n]
    rmax = int(ranks.max()) + 1
    o = order.cpu().numpy()[:rmax]
    rc = rects.cpu().numpy()[o]
    ok = rc[:, 0] >= 0
    nt = np.where(ok, (rc[:, 2] - rc[:, 0] + 1) * (rc[:, 3] - rc[:, 1] + 1), 0)
    hits = np.bincount(ranks, minlength=rmax)
    print(f"pairs {n}  ranks in the phase {rmax}  with a rect {ok.sum()}")
    print(f"candidate tiles {nt.sum()}  hits {hits.sum()}  hit rate {hits.sum() / max(nt.sum(), 1):.3f}")
    for lo, hi in [(1, 1), (2, 4), (5, 16), (17, 64), (65, 256), (257, 10**9)]:
        m = (nt >= lo) & (nt <= hi)
        print(f"  rect {lo:4d}-{hi:<10d} ranks {m.sum():8d}  candidates {nt[m].sum():9d}")
    lanes32 = (np.ceil(nt / 32) * 32).sum()
    print(f"warp-per-rank lane efficiency {nt.sum() / max(lanes32, 1):.3f} "
          f"(issue slots ~ {np.ceil(nt / 32).sum():.0f} warp-iterations)")
    print(f"load-balanced: ~{np.ceil(nt.sum() / 32):.0f} warp-iterations")


if __name__ == "__main__":
    main()

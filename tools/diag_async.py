"""Replay the device-sized first-phase plan of
tests/test_gpu_parity.py::test_device_sized_first_phase_matches_fresh_views
step by step (diagnostics; run under compute-sanitizer)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import oracle.splat_oracle as O  # noqa: E402
from paper_2603_02887_b200 import DeviceScene, _native, backward_device, forward_device  # noqa
from paper_2603_02887_b200.transmittance import TransmittanceModel  # noqa: E402

MODELS = {"softplus_20": TransmittanceModel.softplus(20.0), "linear": TransmittanceModel.linear(),
          "exponential": TransmittanceModel.exponential()}
sc_a = O.round_scene_f32(O.canonical_scene(60_000, seed=2))
sc_b = O.round_scene_f32(O.canonical_scene(90_000, seed=3))
cams = [O.canonical_camera(320, 240, v, 8) for v in (0, 0, 3)]
wide = O.look_at([0, 0, -1.0], [0, 0, 4.0], [0, 1, 0], 80.0, 320, 240)
seed = torch.as_tensor(O.canonical_seed(320, 240, 0), dtype=torch.float32).cuda()


def dev_of(sc):
    return DeviceScene.from_arrays(sc)


dev_a, dev_b = dev_of(sc_a), dev_of(sc_b)
plan = [(dev_a, cams[0], "softplus_20"), (dev_a, cams[1], "softplus_20"),
        (dev_a, wide, "softplus_20"), (dev_a, cams[2], "softplus_20"),
        (dev_b, cams[2], "softplus_20"), (dev_b, cams[2], "linear"),
        (dev_a, cams[0], "exponential"), (dev_a, cams[0], "exponential")]
view = _native.View()
for i, (dev, cam, name) in enumerate(plan):
    print("step", i, name, flush=True)
    out = forward_device(view, dev, cam, MODELS[name], np.zeros(3))
    g = backward_device(view, dev, seed)
    torch.cuda.synchronize()
    print("  ok", view.stats()["n_pairs"], flush=True)

import os, sys, subprocess
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2603_02887_b200 import DeviceScene, _native, backward_device, forward_device
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed
from paper_2603_02887_b200.transmittance import TransmittanceModel
dev = DeviceScene.from_arrays(canonical_scene(1_000_000, seed=5))
cam = canonical_camera(1920, 1080)
seed = torch.as_tensor(canonical_seed(1920, 1080, 0), dtype=torch.float32, device="cuda")
m = TransmittanceModel.softplus(20.0)
view = _native.View()
for i in range(6):
    if i == 5:
        os.environ["NXS_TRACE"] = "1"
        sys.stderr.flush()
    forward_device(view, dev, cam, m, np.zeros(3), chunk_size=1)
    backward_device(view, dev, seed)
torch.cuda.synchronize()

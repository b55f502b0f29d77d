import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2603_02887_b200 import DeviceScene, _native, forward_device
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene
from paper_2603_02887_b200.transmittance import TransmittanceModel
for P, W, H in [(1_000_000, 1920, 1080), (5_000_000, 3840, 2160)]:
    dev = DeviceScene.from_arrays(canonical_scene(P, seed=5))
    for name, m in [("softplus", TransmittanceModel.softplus(20.0)), ("exp", TransmittanceModel.exponential())]:
        view = _native.View()
        forward_device(view, dev, canonical_camera(W, H), m, np.zeros(3), chunk_size=1)
        nt = ((W + 15) // 16) * ((H + 15) // 16)
        rg = torch.zeros((nt, 2), dtype=torch.int32, device="cuda")
        view.binning_export(ranges=rg)
        c = (rg[:, 1] - rg[:, 0]).cpu().numpy()
        q = np.percentile(c, [50, 90, 99, 99.9, 100])
        print(P, name, "pairs", c.sum(), "seg pct50/90/99/99.9/max", q, "sum n^2", (c.astype(np.float64)**2).sum() / 1e6, "M", "n>1024:", (c > 1024).sum(), "n>4096:", (c > 4096).sum(), flush=True)

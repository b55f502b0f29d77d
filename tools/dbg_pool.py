import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2603_02887_b200 import DeviceScene, TransmittanceModel, _native, forward_backward_device
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed
arrs = canonical_scene(1_000_000, seed=5); dev = DeviceScene.from_arrays(arrs)
cams = [canonical_camera(1920, 1080, v, 8) for v in range(8)]
seed = torch.as_tensor(canonical_seed(1920, 1080, 0), dtype=torch.float32).cuda()
m = TransmittanceModel.softplus(20.0)
view = _native.View()
for it in range(2):
    for v in range(8):
        print("== call", it, v, file=sys.stderr, flush=True)
        forward_backward_device(view, dev, cams[v], m, np.zeros(3), seed)
        torch.cuda.synchronize()
print(view.stats())

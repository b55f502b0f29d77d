"""One small forward+backward per ordering mode through the C-ABI, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).
usage: compute-sanitizer --tool T python tools/sanitize_case.py [n W H]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2603_02887_b200 import DeviceScene, _native, forward_backward_device  # noqa: E402
from paper_2603_02887_b200 import TransmittanceModel  # noqa: E402
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed  # noqa

n, W, H = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (20_000, 96, 64)
arrs = canonical_scene(n, seed=5)
dev = DeviceScene.from_arrays(arrs)
cam = canonical_camera(W, H, 1, 8)
seed = torch.as_tensor(canonical_seed(W, H, 1), dtype=torch.float32).cuda()
for model in (TransmittanceModel.softplus(20.0), TransmittanceModel.exponential()):
    for cs in (1, None, 64):
        view = _native.View()
        for _ in range(2):  # second call: device-sized first phase (CUDA graph)
            out, g = forward_backward_device(view, dev, cam, model, np.zeros(3), seed,
                                             chunk_size=cs)
        torch.cuda.synchronize()
        print(model.variant, cs, float(out[0].sum()), float(g["opacities"].abs().sum()),
              flush=True)
        view.close()
print("ok")

"""Exact-order (Mode X) pending-buffer statistics at C3 from the xstats
variant (python -m paper_2603_02887_b200.build --variant=xstats -DNXS_XSTATS)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["NXS_LIB"] = str(ROOT / "paper_2603_02887_b200/lib/libnxs_xstats.so")
import torch  # noqa: E402

from paper_2603_02887_b200 import DeviceScene, TransmittanceModel, _native, forward_device  # noqa
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene  # noqa: E402

arrs = canonical_scene(1_000_000, seed=5)
dev = DeviceScene.from_arrays(arrs)
cam = canonical_camera(1920, 1080)
view = _native.View()
forward_device(view, dev, cam, TransmittanceModel.softplus(20.0), np.zeros(3), chunk_size=None)
torch.cuda.synchronize()
out = (C.c_ulonglong * 40)()
_native.lib().nxs_debug_xstats(out)
v = list(out)
print("inserts", v[0], "shifted", v[1], "mean shift", v[1] / max(1, v[0]), "mean pending",
      v[2] / max(1, v[0]), "commits", v[3])
print("pending-at-insert histogram", v[5:37])

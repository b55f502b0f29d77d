import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2603_02887_b200 as nx
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed
arrs = canonical_scene(1_000_000, seed=5)
cam = canonical_camera(1920, 1080)
seed = canonical_seed(1920, 1080)
m = nx.TransmittanceModel.softplus(20.0)
ts = []
for i in range(10):
    t0 = time.perf_counter(); r = nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=None); ts.append((time.perf_counter()-t0)*1e3)
print("softX", [round(x,1) for x in ts], flush=True)
out = nx.render(arrs, cam, m, np.zeros(3))
print("render ok", out.rgb.shape, flush=True)

import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2603_02887_b200 as nx
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed
arrs = canonical_scene(1_000_000, seed=5)
cam = canonical_camera(1920, 1080)
seed = canonical_seed(1920, 1080)
for name, m, ch in [("exp", nx.TransmittanceModel.exponential(), 1), ("soft", nx.TransmittanceModel.softplus(20.0), 1), ("softX", nx.TransmittanceModel.softplus(20.0), None)]:
    ts = []
    for i in range(6):
        t0 = time.perf_counter(); r = nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=ch); ts.append((time.perf_counter()-t0)*1e3)
    print(name, [round(x,1) for x in ts], flush=True)

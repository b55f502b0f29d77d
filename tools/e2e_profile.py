import sys, time, cProfile, pstats
from pathlib import Path
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2603_02887_b200 as nx
from paper_2603_02887_b200.scenes import canonical_camera, canonical_scene, canonical_seed
arrs = canonical_scene(1_000_000, seed=5)
cam = canonical_camera(1920, 1080)
seed = canonical_seed(1920, 1080)
m = nx.TransmittanceModel.softplus(20.0)
for _ in range(3):
    r = nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=1)
torch.cuda.synchronize()
ts = []
for _ in range(8):
    t0 = time.perf_counter(); r = nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=1); ts.append((time.perf_counter()-t0)*1e3)
print("calls ms", [round(x,2) for x in ts])
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    r = nx.render_with_gradients(arrs, cam, m, np.zeros(3), seed, chunk_size=1)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

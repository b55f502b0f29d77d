import importlib, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
R = importlib.import_module("paper_2603_02887_b200.render")
shapes = {"centers": (1_000_000, 3), "scales": (1_000_000, 3), "quats": (1_000_000, 4),
          "opacities": (1_000_000,), "sh": (1_000_000, 3, 4)}
g = {k: torch.rand(s, device="cuda") for k, s in shapes.items()}
for piece in (1 << 18, 1 << 20, 1 << 22, 1 << 30):
    R._PIECE = piece
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        dl = R._Download()
        for k, v in g.items():
            dl.add(v, "g_" + k)
        t1 = time.perf_counter()
        out = dl.result()
        t2 = time.perf_counter()
    print(f"piece {piece}: queue {1e3*(t1-t0):.2f} ms, result {1e3*(t2-t1):.2f} ms")
host = np.random.rand(23_000_000)
for piece in (1 << 18, 1 << 20, 1 << 22, 1 << 30):
    R._PIECE = piece
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d = R._h2d_f32(host, torch.device("cuda"), "x")
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"piece {piece}: upload {1e3*(t1-t0):.2f} ms")

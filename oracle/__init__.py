"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Checkers for the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` legs may import
this package; the product package ``paper_2603_02887_b200`` never does.

* ``splat_oracle``  — float64 numpy restatement of the reference renderer
  (forward + unified-adjoint backward), pinned to golden vectors produced
  by the reference itself (tests/golden/).
* ``binning_oracle.c`` (via :func:`binning`) — C restatement of the fp64
  projection and tile binning, the bit-exact checker for the device's
  records, tile rectangles, depth order and per-tile lists.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libnxs_oracle.so"


def build_c() -> Path:
    src = HERE / "binning_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build_c()
        h = C.CDLL(str(LIB))
        f = h.nxs_oracle_binning
        f.restype = C.c_int64
        f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                      C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_int64]
        _lib = h
    return _lib


def binning(scene, cam, cutoff=1.0 / 255.0, near=1e-4) -> dict:
    """Run the C restatement on float32 scene arrays; returns order,
    records (P, 32) float32, rects (P, 4), ranges (T, 2), pairs."""
    h = _load()
    f32 = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.float32))  # noqa: E731
    cen, sca, qua, opa = f32(scene.centers), f32(scene.scales), f32(scene.quats), \
        f32(scene.opacities)
    P = len(opa)
    o = np.ascontiguousarray(np.asarray(cam.position, dtype=np.float64).reshape(3))
    R = np.ascontiguousarray(np.asarray(cam.rotation, dtype=np.float64).reshape(9))
    W, H = int(cam.width), int(cam.height)
    T = ((W + 15) // 16) * ((H + 15) // 16)
    order = np.zeros(max(P, 1), np.int32)
    records = np.zeros((max(P, 1), 32), np.float32)
    rects = np.zeros((max(P, 1), 4), np.int32)
    ranges = np.zeros((T, 2), np.int32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    args = (P, p(cen), p(sca), p(qua), p(opa), p(o), p(R), float(cam.focal), float(cam.cx),
            float(cam.cy), W, H, float(cutoff), float(near), p(order), p(records), p(rects),
            p(ranges))
    n = h.nxs_oracle_binning(*args, None, 0)
    if n < 0:
        raise ValueError("a Gaussian straddles the near plane")
    pairs = np.zeros(max(n, 1), np.int32)
    h.nxs_oracle_binning(*args, p(pairs), n)
    return dict(order=order[:P], records=records[:P], rects=rects[:P], ranges=ranges,
                pairs=pairs[:n], n_pairs=int(n), tiles_x=(W + 15) // 16)


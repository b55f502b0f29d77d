"""ctypes binding of the C-ABI library ``lib/libnxs.so`` (include/nxs.h).

This is the only way the package reaches the device: there is no CPU
fallback.  Loading fails loudly (``NativeLibraryError``) when the library
has not been built (``python -m paper_2603_02887_b200.build``) and every
non-zero status code from the library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

__all__ = [
    "NativeLibraryError",
    "NxsError",
    "lib",
    "View",
    "SYMBOLS",
    "make_camera",
    "make_model",
    "make_opts",
]

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libnxs.so"

# every entry point declared in include/nxs.h
SYMBOLS = (
    "nxs_abi_version",
    "nxs_error_string",
    "nxs_last_error",
    "nxs_view_create",
    "nxs_view_destroy",
    "nxs_view_stats",
    "nxs_view_bytes",
    "nxs_view_timings",
    "nxs_view_set_timing",
    "nxs_forward",
    "nxs_backward",
    "nxs_forward_backward",
    "nxs_cache_export",
    "nxs_depth_order",
    "nxs_binning_export",
    "nxs_records_export",
    "nxs_touched_export",
    "nxs_touched_mark",
    "nxs_view_history_bytes",
    "nxs_view_history_save",
    "nxs_view_history_load",
    "nxs_grads_zero_masked",
    "nxs_grads_select",
    "nxs_grads_gather",
    "nxs_grads_scatter",
    "nxs_loss_workspace_bytes",
    "nxs_image_loss",
    "nxs_adam_step",
    "nxs_adam_step_f64",
    "nxs_composite_batch",
)

NXS_ERR_GEOMETRY = -6
NXS_ERR_OVERFLOW = -7
NXS_ERR_UNSUPPORTED = -2
NXS_ERR_INVALID = -1
NXS_FLAG_COUNT_EVENTS = 1
NXS_FLAG_FULL_BINNING = 2
NXS_FLAG_XBUF32 = 4
NXS_FLAG_THETA0 = 8
NXS_FLAG_DETERMINISTIC = 16
NXS_LOSS_SRGB_INPUT = 1


class NativeLibraryError(ImportError):
    pass


class NxsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"nxs error {code}: {msg}")
        self.code = code


class Model(C.Structure):
    _fields_ = [("variant", C.c_int32), ("param", C.c_double)]


class Camera(C.Structure):
    _fields_ = [
        ("position", C.c_double * 3),
        ("rotation", C.c_double * 9),
        ("focal", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


class Opts(C.Structure):
    _fields_ = [
        ("max_splats", C.c_int32),
        ("alpha_cutoff", C.c_double),
        ("near_plane", C.c_double),
        ("chunk_size", C.c_int32),
        ("flags", C.c_int32),
        ("first_phase_ranks", C.c_int64),
    ]


class Scene(C.Structure):
    _fields_ = [
        ("centers", C.c_void_p),
        ("scales", C.c_void_p),
        ("quats", C.c_void_p),
        ("opacities", C.c_void_p),
        ("sh", C.c_void_p),
        ("count", C.c_int64),
        ("sh_coeffs", C.c_int32),
    ]


class AdamGroup(C.Structure):
    _fields_ = [("param", C.c_void_p), ("grad", C.c_void_p), ("m", C.c_void_p),
                ("v", C.c_void_p), ("count", C.c_int64), ("lr", C.c_double)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_gaussians", "n_visible", "n_pairs", "n_straddling", "n_tiles", "n_tests_fwd",
        "n_composited", "n_tests_bwd", "n_entries_bwd", "n_overflow", "n_launches", "n_redo")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


_lib = None


def lib():
    """Load (once) and return the ctypes handle; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("NXS_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not found: build the CUDA library first "
            "(python -m paper_2603_02887_b200.build). There is no CPU fallback.")
    h = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    h.nxs_abi_version.restype = C.c_int
    h.nxs_error_string.restype = C.c_char_p
    h.nxs_error_string.argtypes = [C.c_int]
    h.nxs_last_error.restype = C.c_char_p
    h.nxs_view_create.argtypes = [C.POINTER(vp)]
    h.nxs_view_destroy.argtypes = [vp]
    h.nxs_view_stats.argtypes = [vp, C.POINTER(Stats)]
    h.nxs_view_bytes.argtypes = [vp]
    h.nxs_view_bytes.restype = i64
    h.nxs_view_timings.argtypes = [vp, C.POINTER(C.c_float), C.c_int]
    h.nxs_view_set_timing.argtypes = [vp, C.c_int]
    h.nxs_forward.argtypes = [vp, C.POINTER(Scene), C.POINTER(Camera), C.POINTER(Model),
                              C.POINTER(Opts), C.POINTER(C.c_float), vp, vp, vp, vp]
    h.nxs_backward.argtypes = [vp, C.POINTER(Scene), vp, vp, vp, vp, vp, vp, vp]
    h.nxs_forward_backward.argtypes = [vp, C.POINTER(Scene), C.POINTER(Camera), C.POINTER(Model),
                                       C.POINTER(Opts), C.POINTER(C.c_float), vp, vp, vp, vp,
                                       vp, vp, vp, vp, vp, vp]
    h.nxs_cache_export.argtypes = [vp, vp, vp, vp, vp, vp]
    h.nxs_depth_order.argtypes = [vp, vp, vp]
    h.nxs_binning_export.argtypes = [vp, vp, vp, vp, vp]
    h.nxs_records_export.argtypes = [vp, vp, vp]
    h.nxs_touched_export.argtypes = [vp, vp, C.POINTER(C.c_int64), vp]
    h.nxs_touched_mark.argtypes = [vp, vp, vp]
    h.nxs_view_history_bytes.restype = i64
    h.nxs_view_history_bytes.argtypes = []
    h.nxs_view_history_save.argtypes = [vp, vp]
    h.nxs_view_history_load.argtypes = [vp, vp]
    h.nxs_grads_zero_masked.argtypes = [vp, i64, i32, vp, vp]
    h.nxs_grads_select.argtypes = [vp, i64, vp, C.POINTER(C.c_int64), vp]
    h.nxs_grads_gather.argtypes = [vp, i64, i32, vp, i64, vp, vp]
    h.nxs_grads_scatter.argtypes = [vp, i64, i32, vp, i64, vp, vp]
    h.nxs_loss_workspace_bytes.argtypes = [i32, i32]
    h.nxs_loss_workspace_bytes.restype = i64
    h.nxs_image_loss.argtypes = [vp, vp, i32, i32, C.c_double, i32, vp, vp, vp, vp]
    h.nxs_adam_step.argtypes = [C.POINTER(AdamGroup), i64, C.c_double, vp, vp]
    h.nxs_adam_step_f64.argtypes = [C.POINTER(AdamGroup), i64, C.c_double, vp, vp]
    h.nxs_composite_batch.argtypes = [C.POINTER(Model), vp, vp, vp, i64, i64,
                                      C.POINTER(C.c_double), vp, vp, vp, vp, vp, vp, vp, vp, vp]
    for name in SYMBOLS:
        if name not in ("nxs_error_string", "nxs_last_error", "nxs_view_bytes",
                        "nxs_loss_workspace_bytes", "nxs_view_history_bytes"):
            getattr(h, name).restype = C.c_int
    if h.nxs_abi_version() != 2:
        raise NativeLibraryError("libnxs ABI version mismatch")
    _lib = h
    return h


def grads_zero_masked(flat, n, sh_coeffs, mask, stream=None):
    _check(lib().nxs_grads_zero_masked(_ptr(flat), int(n), int(sh_coeffs), _ptr(mask),
                                       _stream_ptr(stream)))


def grads_select(mask, n, index, stream=None) -> int:
    cnt = C.c_int64(0)
    _check(lib().nxs_grads_select(_ptr(mask), int(n), _ptr(index), C.byref(cnt),
                                  _stream_ptr(stream)))
    return int(cnt.value)


def grads_gather(flat, n, sh_coeffs, index, count, packed, stream=None):
    _check(lib().nxs_grads_gather(_ptr(flat), int(n), int(sh_coeffs), _ptr(index), int(count),
                                  _ptr(packed), _stream_ptr(stream)))


def grads_scatter(flat, n, sh_coeffs, index, count, packed, stream=None):
    _check(lib().nxs_grads_scatter(_ptr(flat), int(n), int(sh_coeffs), _ptr(index), int(count),
                                   _ptr(packed), _stream_ptr(stream)))


def _check(code: int):
    if code != 0:
        msg = lib().nxs_last_error().decode() or lib().nxs_error_string(code).decode()
        raise NxsError(code, msg)


def make_camera(cam) -> Camera:
    c = Camera()
    pos = np.asarray(cam.position, dtype=np.float64).reshape(3)
    rot = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    c.position[:] = [float(x) for x in pos]
    c.rotation[:] = [float(x) for x in rot]
    c.focal, c.cx, c.cy = float(cam.focal), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def make_model(variant_id: int, param: float) -> Model:
    return Model(int(variant_id), float(param))


def make_opts(max_splats, alpha_cutoff, near, chunk_size, flags=0, first_phase_ranks=0) -> Opts:
    cs = 0 if chunk_size is None else int(chunk_size)
    return Opts(int(max_splats), float(alpha_cutoff), float(near), cs, int(flags),
                int(first_phase_ranks))


def _ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def _stream_ptr(stream) -> int | None:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream) or None


class View:
    """Owns one ``nxs_view`` (per-view device workspace + replay cache)."""

    def __init__(self):
        h = lib()
        p = C.c_void_p()
        _check(h.nxs_view_create(C.byref(p)))
        self._p = p
        self._h = h

    def close(self):
        if getattr(self, "_p", None) is not None and self._p.value:
            self._h.nxs_view_destroy(self._p)
            self._p = None

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def scene_struct(dev) -> Scene:
        return Scene(_ptr(dev.centers), _ptr(dev.scales), _ptr(dev.quats), _ptr(dev.opacities),
                     _ptr(dev.sh), int(dev.count), int(dev.sh_coeffs))

    def forward(self, dev, cam: Camera, model: Model, opts: Opts, bg, rgb, overdraw, residual,
                stream=None):
        sc = self.scene_struct(dev)
        bgc = (C.c_float * 3)(*[float(x) for x in bg])
        _check(self._h.nxs_forward(self._p, C.byref(sc), C.byref(cam), C.byref(model),
                                   C.byref(opts), bgc, _ptr(rgb), _ptr(overdraw), _ptr(residual),
                                   _stream_ptr(stream)))

    def backward(self, dev, seed, grads, stream=None):
        sc = self.scene_struct(dev)
        _check(self._h.nxs_backward(self._p, C.byref(sc), _ptr(seed), _ptr(grads["centers"]),
                                    _ptr(grads["scales"]), _ptr(grads["quats"]),
                                    _ptr(grads["opacities"]), _ptr(grads["sh"]),
                                    _stream_ptr(stream)))

    def forward_backward(self, dev, cam: Camera, model: Model, opts: Opts, bg, rgb, overdraw,
                         residual, seed, grads, stream=None):
        sc = self.scene_struct(dev)
        bgc = (C.c_float * 3)(*[float(x) for x in bg])
        _check(self._h.nxs_forward_backward(
            self._p, C.byref(sc), C.byref(cam), C.byref(model), C.byref(opts), bgc, _ptr(rgb),
            _ptr(overdraw), _ptr(residual), _ptr(seed), _ptr(grads["centers"]),
            _ptr(grads["scales"]), _ptr(grads["quats"]), _ptr(grads["opacities"]),
            _ptr(grads["sh"]), _stream_ptr(stream)))

    def cache_export(self, sat=None, e_k=None, t_k=None, theta0=None, stream=None):
        _check(self._h.nxs_cache_export(self._p, _ptr(sat), _ptr(e_k), _ptr(t_k), _ptr(theta0),
                                        _stream_ptr(stream)))

    def depth_order(self, out, stream=None):
        _check(self._h.nxs_depth_order(self._p, _ptr(out), _stream_ptr(stream)))

    def binning_export(self, rects=None, ranges=None, pair_ranks=None, stream=None):
        _check(self._h.nxs_binning_export(self._p, _ptr(rects), _ptr(ranges), _ptr(pair_ranks),
                                          _stream_ptr(stream)))

    def records_export(self, out, stream=None):
        _check(self._h.nxs_records_export(self._p, _ptr(out), _stream_ptr(stream)))

    def history_save(self) -> bytes:
        """The view's sizing history (opaque; see nxs_view_history_save)."""
        buf = C.create_string_buffer(int(self._h.nxs_view_history_bytes()))
        _check(self._h.nxs_view_history_save(self._p, buf))
        return buf.raw

    def history_load(self, blob: bytes):
        _check(self._h.nxs_view_history_load(self._p, C.c_char_p(blob)))

    def touched_mark(self, mask, stream=None):
        """mask[g] = 1 for the Gaussians the last backward wrote (async)."""
        _check(self._h.nxs_touched_mark(self._p, _ptr(mask), _stream_ptr(stream)))

    def touched_export(self, out=None, stream=None) -> int:
        """Gaussians the last backward wrote (into ``out``, int32 CUDA with
        capacity >= the scene count, unless None); returns their number."""
        n = C.c_int64(0)
        _check(self._h.nxs_touched_export(self._p, _ptr(out), C.byref(n), _stream_ptr(stream)))
        return int(n.value)

    def stats(self) -> dict:
        st = Stats()
        _check(self._h.nxs_view_stats(self._p, C.byref(st)))
        return st.as_dict()

    PHASES = ("depth_sort", "project", "binning", "blend_fwd", "n_depth_phases",
              "fwd_bwd_gap", "forward_total", "moment_clear", "blend_bwd", "chain")

    def set_timing(self, on: bool = True) -> "View":
        """Record per-phase CUDA events from the next call on (off by
        default: every event costs the device pipeline a few microseconds)."""
        _check(self._h.nxs_view_set_timing(self._p, 1 if on else 0))
        return self

    def timings(self) -> dict:
        """Device milliseconds per phase of the last forward/backward
        (needs :meth:`set_timing`)."""
        arr = (C.c_float * len(self.PHASES))()
        _check(self._h.nxs_view_timings(self._p, arr, len(self.PHASES)))
        return {n: float(arr[i]) for i, n in enumerate(self.PHASES) if not n.startswith("_")}

    def nbytes(self) -> int:
        return int(self._h.nxs_view_bytes(self._p))

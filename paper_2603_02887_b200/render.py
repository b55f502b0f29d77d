"""Drop-in replacement for the reference module ``nexsplat.render``.

Same names, signatures, argument meaning, return types and error
behaviour as reference ``pkg/src/nexsplat/render.py`` (``__all__`` at
render.py:34-41):

    render(scene, camera, model, background, *, max_splats=128,
           alpha_cutoff=1/255, near=1e-4, chunk_size=None, threads=1)
        -> RenderResult(rgb (H,W,3) f64, overdraw (H,W) int64, residual (H,W) f64)
    render_forward_cached(arrs, camera, model, background, *, ...) -> (RenderResult, cache)
    render_backward(arrs, camera, model, background, cache, seed_image, *, ...) -> grads
    render_with_gradients(arrs, camera, model, background, seed_image, *, ...)

All arithmetic runs in the CUDA library (libnxs, include/nxs.h) on the
current torch CUDA device; this module only moves arrays.  Inputs may be
the reference's numpy ``SceneArrays`` / primitive lists (float64, copied to
the device as float32 each call — the reference mutates them in place
between calls, optimizer.py:382) or a :class:`DeviceScene` of resident
float32 CUDA tensors (the fast path; nothing crosses PCIe but the outputs).

Ordering (reference render.py:171, 350-358), all on the
device: the default ``chunk_size=None`` (exact per-pixel order by peak
depth, "Mode X"), ``chunk_size=1`` (global front-to-back order, "Mode G")
and ``chunk_size=C`` (chunks of C Gaussians in centre-depth order, per-pixel
peak-depth order within each chunk, "Mode C" — the training default
C=128).  A pixel whose pending buffer overflows in the t-ordered modes makes
the call raise ``RuntimeError`` rather than return an unguaranteed order.
"""
from __future__ import annotations

import threading
import weakref
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import _native
from .camera import ALPHA_MAX, DEFAULT_ALPHA_CUTOFF, NEAR_PLANE, GaussianPrimitive
from .transmittance import VARIANT_IDS, as_model

__all__ = [
    "SceneArrays",
    "RenderResult",
    "DeviceScene",
    "render",
    "render_forward_cached",
    "render_backward",
    "render_with_gradients",
    "forward_device",
    "backward_device",
    "zero_grads_device",
]


@dataclass
class SceneArrays:
    """Structure-of-arrays scene (reference render.py:44-87)."""

    centers: np.ndarray   # (P, 3)
    scales: np.ndarray    # (P, 3)
    quats: np.ndarray     # (P, 4), normalised on use
    opacities: np.ndarray  # (P,)
    sh: np.ndarray        # (P, 3, C)

    @classmethod
    def from_primitives(cls, scene) -> "SceneArrays":
        n = len(scene)
        c = max((p.sh.shape[1] for p in scene), default=1)
        sh = np.zeros((n, 3, c))
        for i, p in enumerate(scene):
            sh[i, :, : p.sh.shape[1]] = p.sh
        return cls(
            centers=np.array([p.center for p in scene], dtype=np.float64).reshape(n, 3),
            scales=np.array([p.scale for p in scene], dtype=np.float64).reshape(n, 3),
            quats=np.array([p.rotation for p in scene], dtype=np.float64).reshape(n, 4),
            opacities=np.array([p.opacity for p in scene], dtype=np.float64),
            sh=sh,
        )

    def to_primitives(self) -> list:
        prims = []
        for i in range(len(self.opacities)):
            q = self.quats[i] / np.linalg.norm(self.quats[i])
            prims.append(GaussianPrimitive(
                self.centers[i].copy(), np.maximum(self.scales[i], 1e-6), q,
                float(np.clip(self.opacities[i], 1e-4, ALPHA_MAX)), self.sh[i].copy()))
        return prims

    def __len__(self) -> int:
        return len(self.opacities)

    def copy(self) -> "SceneArrays":
        return SceneArrays(self.centers.copy(), self.scales.copy(), self.quats.copy(),
                           self.opacities.copy(), self.sh.copy())


@dataclass
class RenderResult:
    rgb: np.ndarray       # (H, W, 3) linear radiance
    overdraw: np.ndarray  # (H, W) splats evaluated per pixel
    residual: np.ndarray  # (H, W) transmittance left after all splats


class DeviceScene:
    """Resident float32 CUDA copy of a scene (the B200 fast path)."""

    FIELDS = ("centers", "scales", "quats", "opacities", "sh")

    def __init__(self, centers, scales, quats, opacities, sh):
        import torch
        self.centers = centers.contiguous()
        self.scales = scales.contiguous()
        self.quats = quats.contiguous()
        self.opacities = opacities.contiguous()
        self.sh = sh.contiguous()
        for name in self.FIELDS:
            t = getattr(self, name)
            if t.dtype != torch.float32 or not t.is_cuda:
                raise TypeError(f"DeviceScene.{name} must be a float32 CUDA tensor")
        self.count = int(self.opacities.shape[0])
        self.sh_coeffs = int(self.sh.shape[2]) if self.sh.ndim == 3 else 1
        if self.sh_coeffs not in (1, 4):
            raise ValueError("sh must have 1 or 4 coefficients per channel")

    @classmethod
    def from_arrays(cls, arrs, device=None, non_blocking=False) -> "DeviceScene":
        import torch
        dev = torch.device("cuda") if device is None else torch.device(device)

        def up(x, shape, key):
            if isinstance(x, torch.Tensor):
                return x.to(device=dev, dtype=torch.float32).reshape(shape)
            return _h2d_f32(np.asarray(x).reshape(shape), dev, key)

        n = len(arrs.opacities)
        sh = arrs.sh
        c = int(np.shape(sh)[2]) if len(np.shape(sh)) == 3 else 1
        return cls(up(arrs.centers, (n, 3), "centers"), up(arrs.scales, (n, 3), "scales"),
                   up(arrs.quats, (n, 4), "quats"), up(arrs.opacities, (n,), "opacities"),
                   up(sh, (n, 3, c), "sh"))

    def __len__(self):
        return self.count


# --- host <-> device staging for the numpy API ------------------------------
# float64 numpy in, float64 numpy out (the reference's types).  Transfers are
# pipelined in pieces through cached page-locked buffers: the host converts
# piece k+1 (multi-threaded torch copy) while the DMA engine moves piece k,
# and downloads convert each piece as soon as its copy event fires.
_PIECE = 1 << 22  # elements per pipelined piece (measured: 1M pieces cost 2x on downloads)
_STAGES: dict = {}


class _Stage:
    """A cached page-locked buffer and the event of the last copy using it."""

    def __init__(self, n, dtype):
        import torch
        self.buf = torch.empty(n, dtype=dtype, pin_memory=True)
        self.ev = torch.cuda.Event()
        self.ev.record()
        self.lock = threading.Lock()  # one host thread fills the buffer at a time


_STAGES_LOCK = threading.Lock()


def _stage(key, n, dtype) -> _Stage:
    with _STAGES_LOCK:
        st = _STAGES.get(key)
        if st is None or st.buf.numel() < n or st.buf.dtype != dtype:
            st = _Stage(max(n, 1), dtype)
            _STAGES[key] = st
        return st


def _h2d_f32(a: np.ndarray, dev, key):
    """float64 (or float32) numpy array -> new float32 CUDA tensor."""
    import torch
    src = torch.from_numpy(np.ascontiguousarray(a).reshape(-1))
    n = src.numel()
    out = torch.empty(n, dtype=torch.float32, device=dev)
    st = _stage(("h2d", key), n, torch.float32)
    with st.lock:
        st.ev.synchronize()  # the previous upload from this buffer has left it
        for off in range(0, n, _PIECE):
            end = min(n, off + _PIECE)
            st.buf[off:end].copy_(src[off:end])
            out[off:end].copy_(st.buf[off:end], non_blocking=True)
        st.ev.record(torch.cuda.current_stream(dev))
    return out.reshape(np.shape(a))


class _PinnedPool:
    """Page-locked host buffers handed out as the returned numpy arrays and
    taken back when an array is garbage collected (weakref finalizer): a
    loop that keeps last call's results alive simply holds two sets."""

    def __init__(self):
        self.free: dict = {}
        self.lock = threading.Lock()

    def array(self, shape, dtype):
        import torch
        key = (tuple(shape), dtype)
        with self.lock:
            lst = self.free.get(key)
            t = lst.pop() if lst else None
        if t is None:
            t = torch.empty(tuple(shape), dtype=dtype, pin_memory=True)
        arr = t.numpy()
        weakref.finalize(arr, self._give, key, t)
        return t, arr

    def _give(self, key, t):
        with self.lock:
            self.free.setdefault(key, []).append(t)


_POOL_PINNED = _PinnedPool()


class _Download:
    """Device -> host results as float64 / int64 numpy arrays.  The widening
    happens on the device and the copy lands directly in page-locked host
    memory that the returned arrays own (recycled through
    :class:`_PinnedPool`): no host-side conversion pass and no first-touch
    page faults."""

    def __init__(self):
        self.items = []

    def add(self, t, key=None):
        import torch
        wide = torch.float64 if t.is_floating_point() else torch.int64
        dev = t.to(wide)
        host, arr = _POOL_PINNED.array(tuple(t.shape), wide)
        host.copy_(dev, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(t.device))
        self.items.append((arr, ev, dev))

    def result(self) -> list:
        outs = []
        for arr, ev, _ in self.items:
            ev.synchronize()
            outs.append(arr)
        self.items = []
        return outs


_SIDE: dict = {}


def _side_stream(dev):
    import torch
    s = _SIDE.get(dev)
    if s is None:
        s = _SIDE[dev] = torch.cuda.Stream(device=dev)
    return s


def _as_device_scene(scene) -> DeviceScene:
    if isinstance(scene, DeviceScene):
        return scene
    if isinstance(scene, (list, tuple)):
        scene = SceneArrays.from_primitives(scene)
    return DeviceScene.from_arrays(scene)


def _effective_chunk(chunk_size, n: int) -> int:
    """Map the reference chunk_size onto the device ordering mode
    (reference render.py:350-354: None or >= P means one exact chunk)."""
    if n <= 1:
        return 1  # every order coincides
    if chunk_size is None or int(chunk_size) >= n:
        return 0
    c = int(chunk_size)
    if c < 1:
        raise ValueError("chunk_size must be >= 1 or None")
    return c


def _check_mode(chunk: int):
    """0: exact per-pixel order, 1: global depth order, C > 1: chunks of C."""
    if chunk < 0:
        raise ValueError("chunk_size must be >= 1 or None")


def _model_struct(model):
    m = as_model(model)
    return m, _native.make_model(VARIANT_IDS[m.variant], m.param)


def _forward_args(dev, camera, model, background, max_splats, alpha_cutoff, near, chunk_size,
                  count_events, full_binning, first_phase_ranks, out, theta0=False,
                  deterministic=False):
    import torch
    chunk = _effective_chunk(chunk_size, dev.count)
    _check_mode(chunk)
    _, ms = _model_struct(model)
    H, W = int(camera.height), int(camera.width)
    d = dev.centers.device
    if out is None:
        out = (torch.empty((H, W, 3), dtype=torch.float32, device=d),
               torch.empty((H, W), dtype=torch.int32, device=d),
               torch.empty((H, W), dtype=torch.float32, device=d))
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    flags = (_native.NXS_FLAG_COUNT_EVENTS if count_events else 0) | \
        (_native.NXS_FLAG_FULL_BINNING if full_binning else 0) | \
        (_native.NXS_FLAG_THETA0 if theta0 else 0) | \
        (_native.NXS_FLAG_DETERMINISTIC if deterministic else 0)
    opts = _native.make_opts(max_splats, alpha_cutoff, near, chunk, flags, first_phase_ranks)
    return _native.make_camera(camera), ms, opts, bg, out


def _raise_mapped(e):
    if e.code == _native.NXS_ERR_OVERFLOW:
        raise RuntimeError(f"{e} (exact order could not be guaranteed)") from e
    if e.code in (_native.NXS_ERR_GEOMETRY, _native.NXS_ERR_UNSUPPORTED):
        raise NotImplementedError(str(e)) from e
    if e.code == _native.NXS_ERR_INVALID:
        raise ValueError(str(e)) from e
    raise e


def forward_device(view, dev: DeviceScene, camera, model, background, *, max_splats=128,
                   alpha_cutoff=DEFAULT_ALPHA_CUTOFF, near=NEAR_PLANE, chunk_size=1,
                   count_events=False, full_binning=False, first_phase_ranks=0, out=None,
                   stream=None, theta0=False, deterministic=False):
    """Forward render on the device; returns (rgb (H,W,3), overdraw (H,W)
    int32, residual (H,W)) float32 CUDA tensors.  ``theta0`` also keeps the
    reference cache's theta0 for :meth:`View.cache_export`;
    ``deterministic`` makes the following backward bit-reproducible
    (NXS_FLAG_DETERMINISTIC, chunk_size=1)."""
    cam, ms, opts, bg, out = _forward_args(dev, camera, model, background, max_splats,
                                           alpha_cutoff, near, chunk_size, count_events,
                                           full_binning, first_phase_ranks, out, theta0,
                                           deterministic)
    try:
        view.forward(dev, cam, ms, opts, bg, out[0], out[1], out[2], stream=stream)
    except _native.NxsError as e:
        _raise_mapped(e)
    return out


def forward_backward_device(view, dev: DeviceScene, camera, model, background, seed, grads=None,
                            *, max_splats=128, alpha_cutoff=DEFAULT_ALPHA_CUTOFF,
                            near=NEAR_PLANE, chunk_size=1, count_events=False,
                            full_binning=False, first_phase_ranks=0, out=None, stream=None,
                            deterministic=False):
    """Forward render plus gradient accumulation for ``seed`` in one library
    call (``nxs_forward_backward``: the end-of-forward depth-phase check
    overlaps the backward).  Returns ((rgb, overdraw, residual), grads).
    ``deterministic``: bit-reproducible gradients (chunk_size=1)."""
    cam, ms, opts, bg, out = _forward_args(dev, camera, model, background, max_splats,
                                           alpha_cutoff, near, chunk_size, count_events,
                                           full_binning, first_phase_ranks, out,
                                           deterministic=deterministic)
    if grads is None:
        grads = zero_grads_device(dev)
    try:
        view.forward_backward(dev, cam, ms, opts, bg, out[0], out[1], out[2], seed.contiguous(),
                              grads, stream=stream)
    except _native.NxsError as e:
        _raise_mapped(e)
    return out, grads


def _same_scene(arrs, dev: DeviceScene) -> bool:
    """``arrs`` (host or device, any float dtype) equals the device scene at
    the device precision (float32), field by field."""
    import torch
    n = dev.count
    for name, shape in (("centers", (n, 3)), ("scales", (n, 3)), ("quats", (n, 4)),
                        ("opacities", (n,)), ("sh", tuple(dev.sh.shape))):
        x = getattr(arrs, name)
        if isinstance(x, torch.Tensor):
            t = x.to(device=dev.centers.device, dtype=torch.float32).reshape(shape)
        else:
            x = np.asarray(x)
            if x.size != int(np.prod(shape)):
                return False
            t = _h2d_f32(x.reshape(shape), dev.centers.device, "cmp_" + name)
        if not torch.equal(t, getattr(dev, name)):
            return False
    return True


def zero_grads_device(dev: DeviceScene) -> dict:
    import torch
    return {
        "centers": torch.zeros_like(dev.centers),
        "scales": torch.zeros_like(dev.scales),
        "quats": torch.zeros_like(dev.quats),
        "opacities": torch.zeros_like(dev.opacities),
        "sh": torch.zeros_like(dev.sh),
    }


def backward_device(view, dev: DeviceScene, seed, grads=None, stream=None) -> dict:
    """Accumulate parameter gradients for ``seed`` (H,W,3 float32 CUDA)
    into ``grads`` (dict of float32 CUDA tensors shaped like the scene)."""
    if grads is None:
        grads = zero_grads_device(dev)
    seed = seed.contiguous()
    view.backward(dev, seed, grads, stream=stream)
    return grads


# Reusable per-view device workspaces for the numpy API (a view grows its
# buffers once and keeps them; allocating ~1 GB per call would dominate).
_POOL: list = []
_POOL_LOCK = threading.Lock()
_POOL_MAX = 4


def _acquire_view():
    with _POOL_LOCK:
        if _POOL:
            return _POOL.pop()
    return _native.View()


def _release_view(view):
    with _POOL_LOCK:
        if len(_POOL) < _POOL_MAX:
            _POOL.append(view)
            return
    view.close()


class _ForwardState:
    """Opaque device state handed from render_forward_cached to
    render_backward (the reference cache is opaque too, render.py:435-436)."""

    def __init__(self, view, dev, settings, outputs):
        self.view, self.dev, self.settings, self.outputs = view, dev, settings, outputs
        weakref.finalize(self, _release_view, view)


class ForwardCache(Mapping):
    """The reference cache dict (render.py:214-217) — keys rad, residual,
    overdraw, sat, e_k, t_k, theta0, flat over pixels, float64 — fetched
    from the device lazily on first access."""

    KEYS = ("rad", "residual", "overdraw", "sat", "e_k", "t_k", "theta0")

    def __init__(self, state: _ForwardState, result: RenderResult):
        self._state = state
        self._result = result
        self._vals: dict = {}

    def _load(self):
        import torch
        st = self._state
        rgb, _, _ = st.outputs
        H, W = rgb.shape[:2]
        d = rgb.device
        sat = torch.empty((H * W,), dtype=torch.uint8, device=d)
        e_k = torch.empty((H * W, 3), dtype=torch.float32, device=d)
        t_k = torch.empty((H * W,), dtype=torch.float32, device=d)
        th0 = torch.empty((H * W, 3), dtype=torch.float32, device=d)
        st.view.cache_export(sat, e_k, t_k, th0)
        r = self._result
        self._vals = {
            "rad": r.rgb.reshape(-1, 3),
            "residual": r.residual.reshape(-1),
            "overdraw": r.overdraw.reshape(-1),
            "sat": sat.cpu().numpy().astype(bool),
            "e_k": e_k.cpu().numpy().astype(np.float64),
            "t_k": t_k.cpu().numpy().astype(np.float64),
            "theta0": th0.cpu().numpy().astype(np.float64),
        }

    def __getitem__(self, key):
        if key == "_nxs":
            return self._state
        if key not in self.KEYS:
            raise KeyError(key)
        if not self._vals:
            self._load()
        return self._vals[key]

    def __iter__(self):
        return iter(self.KEYS)

    def __len__(self):
        return len(self.KEYS)


def _result_to_host(out) -> RenderResult:
    dl = _Download()
    for t, k in zip(out, ("rgb", "overdraw", "residual")):
        dl.add(t, k)
    return RenderResult(*dl.result())


def _settings(camera, model, background, max_splats, alpha_cutoff, near, chunk_size):
    m = as_model(model)
    return (int(camera.width), int(camera.height), float(camera.focal), float(camera.cx),
            float(camera.cy), tuple(np.asarray(camera.position, dtype=np.float64).ravel()),
            tuple(np.asarray(camera.rotation, dtype=np.float64).ravel()), m.variant,
            float(m.param), tuple(np.asarray(background, dtype=np.float64).ravel()),
            int(max_splats), float(alpha_cutoff), float(near),
            None if chunk_size is None else int(chunk_size))


def render(scene, camera, model, background, *, max_splats: int = 128,
           alpha_cutoff: float = DEFAULT_ALPHA_CUTOFF, near: float = NEAR_PLANE,
           chunk_size: int | None = None, threads: int = 1) -> RenderResult:
    """Render radiance, overdraw and residual transmittance (reference
    render.py:361-405).  ``threads`` is accepted and ignored: the output is
    identical for any value, as in the reference."""
    del threads
    background = np.asarray(background, dtype=np.float64)
    dev = _as_device_scene(scene)
    view = _acquire_view()
    try:
        out = forward_device(view, dev, camera, model, background, max_splats=max_splats,
                             alpha_cutoff=alpha_cutoff, near=near, chunk_size=chunk_size)
        return _result_to_host(out)
    finally:
        _release_view(view)


def render_forward_cached(arrs, camera, model, background, *, max_splats: int = 128,
                          alpha_cutoff: float = DEFAULT_ALPHA_CUTOFF, near: float = NEAR_PLANE,
                          chunk_size: int | None = None):
    """Forward sweep plus the replay cache (reference render.py:408-425)."""
    background = np.asarray(background, dtype=np.float64)
    dev = _as_device_scene(arrs)
    view = _acquire_view()
    try:
        out = forward_device(view, dev, camera, model, background, max_splats=max_splats,
                             alpha_cutoff=alpha_cutoff, near=near, chunk_size=chunk_size,
                             theta0=True)
    except BaseException:
        _release_view(view)
        raise
    result = _result_to_host(out)
    st = _ForwardState(view, dev, _settings(camera, model, background, max_splats,
                                            alpha_cutoff, near, chunk_size), out)
    return result, ForwardCache(st, result)


def render_backward(arrs, camera, model, background, cache, seed_image, *,
                    max_splats: int = 128, alpha_cutoff: float = DEFAULT_ALPHA_CUTOFF,
                    near: float = NEAR_PLANE, chunk_size: int | None = None) -> dict:
    """Parameter gradients for an adjoint seed, replaying the traversal that
    produced ``cache`` (reference render.py:428-442).  Settings must match
    the forward call.  Unlike the reference (render.py:229-231) every
    transmittance model has a backward here."""
    import torch
    try:
        st = cache["_nxs"]
    except (KeyError, TypeError):
        raise ValueError("cache was not produced by this package's render_forward_cached")
    if _settings(camera, model, background, max_splats, alpha_cutoff, near,
                 chunk_size) != st.settings:
        raise ValueError("render_backward settings must match the forward call")
    if len(arrs) != st.dev.count:
        raise ValueError("scene size differs from the forward call")
    # The replay runs on the forward's projected scene (the cache describes
    # that traversal); the reference recomputes the geometry from ``arrs``
    # (render.py:437-442), so ``arrs`` must be the forward's scene.
    dev = st.dev
    if arrs is not dev and not _same_scene(arrs, dev):
        raise ValueError("render_backward: arrs differ from the scene of the forward call "
                         "(the cache replays that forward's traversal)")
    H, W = int(camera.height), int(camera.width)
    seed = np.asarray(seed_image, dtype=np.float64).reshape(H, W, 3) if not isinstance(
        seed_image, torch.Tensor) else seed_image
    if isinstance(seed, torch.Tensor):
        seed_t = seed.to(device=dev.centers.device, dtype=torch.float32).contiguous()
    else:
        seed_t = _h2d_f32(seed, dev.centers.device, "seed")
    g = backward_device(st.view, dev, seed_t)
    dl = _Download()
    for k, v in g.items():
        dl.add(v, "g_" + k)
    return dict(zip(g.keys(), dl.result()))


# bytes moved by the last render_with_gradients call (instrumentation, bench.py)
_LAST_IO: dict = {}


def render_with_gradients(arrs, camera, model, background, seed_image, *,
                          max_splats: int = 128, alpha_cutoff: float = DEFAULT_ALPHA_CUTOFF,
                          near: float = NEAR_PLANE, chunk_size: int | None = None):
    """Forward render plus parameter gradients (reference render.py:445-464).

    One fused library call (forward + backward); all results then download
    in pieces that are converted to float64 as they land."""
    import torch
    background = np.asarray(background, dtype=np.float64)
    H, W = int(camera.height), int(camera.width)
    if isinstance(seed_image, torch.Tensor):
        seed = seed_image
    else:
        seed = np.asarray(seed_image, dtype=np.float64).reshape(H, W, 3)
    dev = _as_device_scene(arrs)
    d = dev.centers.device
    view = _acquire_view()
    try:
        if isinstance(seed, torch.Tensor):
            seed_t = seed.to(device=d, dtype=torch.float32).reshape(H, W, 3).contiguous()
        else:
            seed_t = _h2d_f32(seed, d, "seed")
        out, grads = forward_backward_device(view, dev, camera, model, background, seed_t,
                                             max_splats=max_splats, alpha_cutoff=alpha_cutoff,
                                             near=near, chunk_size=chunk_size)
        dl = _Download()
        for t, k in zip(out, ("rgb", "overdraw", "residual")):
            dl.add(t, k)
        # Every gradient row travels, widened to float64 on the device, into
        # recycled page-locked arrays.  Moving only the touched rows (~3 % at
        # C3, nxs_touched_export) was measured slower: the dense float64
        # arrays must then be zero-filled on the host, 184 MB at ~10 ms, vs
        # ~3.4 ms of DMA (profiles/r02_e2e_probe.txt).
        for k, v in grads.items():
            dl.add(v, "g_" + k)
        res = dl.result()
        result = RenderResult(*res[:3])
        g = dict(zip(grads.keys(), res[3:]))
        _LAST_IO.update(d2h=H * W * 5 * 8 + sum(v.numel() for v in grads.values()) * 8)
        _LAST_IO.update(h2d=sum(int(np.prod(np.shape(getattr(arrs, f)))) * 4
                                for f in DeviceScene.FIELDS) + H * W * 3 * 4
                        if not isinstance(arrs, DeviceScene) else H * W * 3 * 4)
    finally:
        _release_view(view)
    return result, g

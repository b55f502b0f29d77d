"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference renderer's forward sweep and
path-replay backward (reference ``pkg/src/nexsplat/render.py:97-358``,
``transmittance.py:215-265``, ``primitives.py:45-93,192-203``).  It is the
checker for the CUDA path: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it.
The product package never imports anything under ``oracle/``.

Parity pinning: ``tests/test_oracle_golden.py`` checks this module against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``): forward images/overdraw/cache for all
models and ordering modes, reference ``render_backward`` gradients for
exponential/linear/quadratic, and reference-forward central finite
differences for softplus and blended (the reference has no analytic
backward for those two, render.py:229-231).

Semantics restated (reference file:line):

* per (Gaussian, pixel) geometry, R3: render.py:109-138
* emission, R4: render.py:97-106, 141-144
* order, R5: render.py:171 (stable per-pixel argsort by t, invalid last),
  render.py:350-358 (chunked global depth order).  Instead of the
  reference's chunk loop we do one per-pixel lexsort on
  (chunk index, t, position-in-chunk) — identical order, since pixels are
  independent and the reference's active-set pruning (render.py:164) only
  drops pixels that are already done.
* per-pixel loop and finalize, R6/R7: render.py:181-217
* weights p̄, R8: transmittance.py:234-262
* backward: the unified adjoint in its fp64 front-to-back
  form; equals reference render.py:288-314 for exp/linear/quadratic and
  extends it to blended/vicini/softplus/power_law.
* chain to parameters: render.py:326-341 (incl. its quaternion projection
  without the 1/|q| factor, render.py:339).

Candidate pruning (``prune=True``) drops (Gaussian, pixel) pairs whose ray
misses the Gaussian's cutoff bounding sphere (radius r·max(s),
r² = 2 ln(ℵ/cutoff)).  Such pairs can never be valid (the kernel peak of a
valid pair lies inside the cutoff ellipsoid), so pruning is exact; it is
only an oracle speed-up.  ``prune=False`` is the reference's brute-force
O(P) per pixel and is what the CPU baseline times.
"""
from __future__ import annotations

import numpy as np

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
ALPHA_MAX = 1.0 - 1e-6
_POWER_LAW_V_EPS = 1e-4

__all__ = [
    "Scene",
    "quat_to_rot",
    "quat_rot_jacobian",
    "pixel_directions",
    "depth_order",
    "forward",
    "backward",
    "render_with_gradients",
    "canonical_scene",
    "canonical_camera",
    "round_scene_f32",
]


class Scene:
    """SoA scene, float64 (same fields as reference SceneArrays, render.py:44-52)."""

    def __init__(self, centers, scales, quats, opacities, sh):
        self.centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
        self.scales = np.asarray(scales, dtype=np.float64).reshape(-1, 3)
        self.quats = np.asarray(quats, dtype=np.float64).reshape(-1, 4)
        self.opacities = np.asarray(opacities, dtype=np.float64).reshape(-1)
        sh = np.asarray(sh, dtype=np.float64)
        c = sh.shape[-1] if sh.ndim == 3 else max(1, sh.size // max(1, 3 * len(self.opacities)))
        self.sh = sh.reshape(len(self.opacities), 3, c)

    @classmethod
    def of(cls, s) -> "Scene":
        return cls(s.centers, s.scales, s.quats, s.opacities, s.sh)

    def __len__(self):
        return len(self.opacities)


# ---------------------------------------------------------------------------
# geometry helpers
# ---------------------------------------------------------------------------

def quat_to_rot(q):
    """reference primitives.py:45-64"""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def quat_rot_jacobian(q):
    """dR/dq at the (unit) point, (..., 4, 3, 3) — reference primitives.py:67-93"""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    o = np.zeros_like(w)
    J = np.empty(q.shape[:-1] + (4, 3, 3))

    def m(rows):
        return np.stack([np.stack(r, -1) for r in rows], -2)

    J[..., 0, :, :] = 2 * m([[o, -z, y], [z, o, -x], [-y, x, o]])
    J[..., 1, :, :] = 2 * m([[o, y, z], [y, -2 * x, -w], [z, w, -2 * x]])
    J[..., 2, :, :] = 2 * m([[-2 * y, x, w], [x, o, z], [-w, z, -2 * y]])
    J[..., 3, :, :] = 2 * m([[-2 * z, -w, x], [w, -2 * z, y], [x, y, o]])
    return J


def pixel_directions(cam):
    """(H*W, 3) unit world directions, reference primitives.py:192-203"""
    j = np.arange(cam.width) + 0.5
    i = np.arange(cam.height) + 0.5
    d = np.empty((cam.height, cam.width, 3))
    d[..., 0] = ((j - cam.cx) / cam.focal)[None, :]
    d[..., 1] = ((i - cam.cy) / cam.focal)[:, None]
    d[..., 2] = 1.0
    R = np.asarray(cam.rotation, dtype=np.float64)
    dw = d @ R.T
    dw /= np.linalg.norm(dw, axis=-1, keepdims=True)
    return dw.reshape(-1, 3)


def sh_basis(dirs, C):
    """reference render.py:97-106"""
    Y = np.empty((dirs.shape[0], C))
    Y[:, 0] = SH_C0
    if C == 4:
        Y[:, 1] = -SH_C1 * dirs[:, 1]
        Y[:, 2] = SH_C1 * dirs[:, 2]
        Y[:, 3] = -SH_C1 * dirs[:, 0]
    return Y


def depth_order(scene, cam):
    """Stable front-to-back order by view depth (μ-o)·forward — reference
    render.py:350-358 (``_depth_chunks`` ordering)."""
    forward = np.asarray(cam.rotation, dtype=np.float64)[:, 2]
    depth = (scene.centers - np.asarray(cam.position, dtype=np.float64)) @ forward
    return np.argsort(depth, kind="stable")


# ---------------------------------------------------------------------------
# transmittance weights
# ---------------------------------------------------------------------------

def _softplus(x):
    return np.logaddexp(0.0, x)


def _expit(x):
    return 0.5 * (1.0 + np.tanh(0.5 * x))


def weight_terms(variant, param, tau, prod):
    """Return (g, fprime, gamma): p̄ = α·g (transmittance.py:234-262).

    τ-family (linear, quadratic, softplus, power_law): g = f(τ̄), f' = df/dτ̄,
    gamma = 0.  P-family (exponential: γ=1; blended/vicini: γ):
    g = (1-γ) + γ·P, fprime unused.
    """
    v = variant
    if v == "exponential":
        return prod, np.zeros_like(tau), 1.0
    if v in ("blended", "vicini"):
        g = param
        if v == "blended":
            gg = 1.0 - g * (1.0 - prod)
        else:
            gg = 1.0 + g * (prod - 1.0)
        return gg, np.zeros_like(tau), g
    if v == "linear":
        return np.ones_like(tau), np.zeros_like(tau), 0.0
    if v == "quadratic":
        c = param
        return 1.0 + c * tau, np.full_like(tau, c), 0.0
    if v == "softplus":
        k = param
        K = k / _softplus(k)
        s = _expit(k * (1.0 - tau))
        f = K * s
        return f, -k * f * (1.0 - s), 0.0
    if v == "power_law":
        w = param
        if w == -1.0:
            return np.ones_like(tau), np.zeros_like(tau), 0.0
        if abs(w) < _POWER_LAW_V_EPS:
            e = np.exp(-tau)
            return e, -e, 0.0
        base = 1.0 + tau * w
        safe = np.where(base > 0.0, base, 1.0)
        ex = -(1.0 + w) / w
        f = np.where(base > 0.0, safe ** ex, 0.0)
        fp = np.where(base > 0.0, ex * w * safe ** (ex - 1.0), 0.0)
        return f, fp, 0.0
    raise ValueError(f"unknown variant {v!r}")


def extinction(variant, param, a, tau, prod):
    """reference transmittance.py:215-265 (discrete_extinction)."""
    if variant == "exponential":
        return a * prod
    if variant == "linear":
        return a * np.ones_like(tau)
    if variant == "quadratic":
        return a * (1.0 + param * tau)
    if variant == "blended":
        return a * (1.0 - param * (1.0 - prod))
    if variant == "vicini":
        lin = a
        ex = a * prod
        return lin + param * (ex - lin)
    if variant == "power_law":
        w = param
        if w == -1.0:
            return a * np.ones_like(tau)
        if abs(w) < _POWER_LAW_V_EPS:
            return a * np.exp(-tau)
        base = 1.0 + tau * w
        safe = np.where(base > 0.0, base, 1.0)
        return a * np.where(base > 0.0, safe ** (-(1.0 + w) / w), 0.0)
    if variant == "softplus":
        k = param
        return a * (k / _softplus(k)) * _expit(k * (1.0 - tau))
    raise ValueError(f"unknown variant {variant!r}")


# ---------------------------------------------------------------------------
# per (row, pixel) geometry
# ---------------------------------------------------------------------------

def _geometry(scene, ids, dirs, origin, near, cutoff):
    """reference render.py:109-138, float64."""
    q = scene.quats[ids]
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    R = quat_to_rot(q)
    s = scene.scales[ids]
    A = np.einsum("rab,rb,rcb->rac", R, 1.0 / s ** 2, R)
    b = scene.centers[ids] - origin[None, :]
    Ad = np.einsum("rac,mc->rma", A, dirs)
    dAd = np.einsum("rma,ma->rm", Ad, dirs)
    bAd = np.einsum("ra,rma->rm", b, Ad)
    t = bAd / dAd
    diff = t[:, :, None] * dirs[None, :, :] - b[:, None, :]
    Adiff = np.einsum("rac,rmc->rma", A, diff)
    m2 = np.einsum("rma,rma->rm", diff, Adiff)
    kernel = np.exp(-0.5 * m2)
    alpha_raw = scene.opacities[ids][:, None] * kernel
    clamped = alpha_raw >= ALPHA_MAX
    alpha = np.minimum(alpha_raw, ALPHA_MAX)
    valid = (t > near) & (alpha >= cutoff)
    return dict(q=q, R=R, s=s, t=t, alpha=alpha, valid=valid, kernel=kernel,
                clamped=clamped, diff=diff, Adiff=Adiff)


def _candidates(scene, dirs, origin, cutoff, prune):
    """Conservative candidate rows for a pixel batch (see module doc)."""
    n = len(scene)
    if not prune:
        return np.arange(n)
    op = scene.opacities
    ok = op >= cutoff
    r = np.sqrt(2.0 * np.log(np.where(ok, op / cutoff, 1.0)))
    rad = r * scene.scales.max(axis=1) * (1.0 + 1e-6) + 1e-12
    b = scene.centers - origin[None, :]
    keep = np.zeros(n, dtype=bool)
    idx = np.nonzero(ok)[0]
    bb = b[idx]
    bn2 = np.einsum("ra,ra->r", bb, bb)
    # distance² from centre to each pixel ray line, in row blocks
    step = max(1, 4_000_000 // max(1, dirs.shape[0]))
    for s0 in range(0, len(idx), step):
        sl = slice(s0, s0 + step)
        proj = bb[sl] @ dirs.T                           # (r, m)
        d2 = bn2[sl, None] - proj * proj
        hit = (d2 <= (rad[idx[sl]] ** 2)[:, None]).any(axis=1)
        keep[idx[sl][hit]] = True
    return np.nonzero(keep)[0]


# ---------------------------------------------------------------------------
# forward
# ---------------------------------------------------------------------------

def _group_keys(scene, cam, chunk_size):
    """Per-Gaussian (group, tie) keys that reproduce the reference order:
    chunk_size None (or >= P): one group, ties by storage index;
    otherwise group = position-in-depth-order // C, tie = depth position."""
    n = len(scene)
    if chunk_size is None or chunk_size >= n:
        return np.zeros(n, dtype=np.int64), np.arange(n, dtype=np.int64)
    order = depth_order(scene, cam)
    pos = np.empty(n, dtype=np.int64)
    pos[order] = np.arange(n)
    return pos // int(chunk_size), pos


def _forward_batch(scene, cam, model, bg, dirs, max_splats, cutoff, near,
                   group, tie, prune):
    variant, param = model.variant, float(getattr(model, "param", 0.0))
    origin = np.asarray(cam.position, dtype=np.float64)
    m = dirs.shape[0]
    ids = _candidates(scene, dirs, origin, cutoff, prune)
    C = scene.sh.shape[2]
    st = dict(ids=ids)
    if ids.size == 0:
        geo = None
    else:
        geo = _geometry(scene, ids, dirs, origin, near, cutoff)
        Y = sh_basis(dirs, C)
        raw = np.einsum("rck,mk->rmc", scene.sh[ids], Y)
        E = np.maximum(raw, 0.0)
        tm = np.where(geo["valid"], geo["t"], np.inf)
        # per-pixel lexsort: group, then t, then tie (stable within chunk)
        g_r = group[ids][:, None] * np.ones((1, m), dtype=np.int64)
        t_r = tie[ids][:, None] * np.ones((1, m), dtype=np.int64)
        # invalid entries go last regardless of group
        g_r = np.where(geo["valid"], g_r, np.iinfo(np.int64).max)
        order = np.lexsort((t_r, tm, g_r), axis=0)
        st.update(geo=geo, Y=Y, E=E, Epos=raw > 0.0, order=order)

    cum = np.zeros(m)
    tau = np.zeros(m)
    prod = np.ones(m)
    count = np.zeros(m, dtype=np.int64)
    rad = np.zeros((m, 3))
    sat = np.zeros(m, dtype=bool)
    e_k = np.broadcast_to(bg, (m, 3)).copy()
    t_k = np.zeros(m)
    sea = np.zeros((m, 3))
    sa = np.zeros(m)
    slots = []  # per slot: (rows, go, satnow, alpha, E, tau_before, prod_before, w)
    # decision margins (SURVEY §8c protocol): distance of any candidate's
    # ln α to ln cutoff, and of any live splat's raw weight to 1 - cum
    amargin = np.full(m, np.inf)
    smargin = np.full(m, np.inf)
    tmargin = np.full(m, np.inf)
    if geo is not None:
        la = np.log(np.maximum(geo["alpha"], 1e-300))
        amargin = np.min(np.abs(la - np.log(cutoff)), axis=0)
        order = st["order"]
        cols = np.arange(m)
        for slot in range(order.shape[0]):
            rows = order[slot]
            a = geo["alpha"][rows, cols]
            val = geo["valid"][rows, cols]
            live = val & ~sat & (count < max_splats)
            if not live.any():
                if not val.any():
                    break  # sorted: no valid entry remains for any pixel
                continue
            e = st["E"][rows, cols]
            w_raw = extinction(variant, param, a, tau, prod)
            sat_now = live & (cum + w_raw >= 1.0)
            go = live & ~sat_now
            w = np.where(sat_now, 1.0 - cum, np.where(go, w_raw, 0.0))
            smargin = np.where(live, np.minimum(smargin, np.abs((1.0 - cum) - w_raw)), smargin)
            slots.append((rows, go, sat_now, a, e, tau.copy(), prod.copy(), w))
            rad += w[:, None] * e
            not_first = count >= 1
            count = count + live
            add = np.where(go, a, 0.0)
            keep = go & not_first
            sea += np.where(keep[:, None], add[:, None] * e, 0.0)
            sa += np.where(keep, add, 0.0)
            cum += np.where(go, w, 0.0)
            tau += add
            prod *= 1.0 - add
            e_k = np.where(sat_now[:, None], e, e_k)
            t_k = np.where(sat_now, w, t_k)
            sat |= sat_now
    if geo is not None and slots:
        # relative gap between consecutive peak depths among the replayed
        # prefix (orders that depend on t: chunk_size None or C > 1)
        order = st["order"]
        k = min(len(slots) + 1, order.shape[0])
        cols = np.arange(m)
        tt = geo["t"][order[:k], cols[None, :]]
        vv = geo["valid"][order[:k], cols[None, :]]
        gi = group[ids][order[:k]] if group is not None else None
        if k >= 2:
            gap = np.abs(np.diff(tt, axis=0)) / np.maximum(np.abs(tt[:-1]), 1e-300)
            ok = vv[1:] & vv[:-1]
            if gi is not None:
                ok &= gi[1:] == gi[:-1]
            gap = np.where(ok, gap, np.inf)
            tmargin = gap.min(axis=0)
    residual = np.where(sat, 0.0, 1.0 - cum)
    rad += bg[None, :] * residual[:, None]
    t_k = np.where(sat, t_k, residual)
    theta0 = sea - e_k * sa[:, None]
    out = dict(rad=rad, residual=residual, overdraw=count, sat=sat, e_k=e_k,
               t_k=t_k, theta0=theta0, tau=tau, prod=prod, cum=cum,
               amargin=amargin, smargin=smargin, tmargin=tmargin)
    st["slots"] = slots
    return out, st


def _pixel_batches(cam, pixels, batch):
    """Group pixel indices into spatially coherent batches (8x8 blocks for
    full images) so pruned candidate unions stay small."""
    W = cam.width
    pixels = np.asarray(pixels, dtype=np.int64)
    r, c = pixels // W, pixels % W
    key = (r // 8) * ((W + 7) // 8) + (c // 8)
    order = np.argsort(key, kind="stable")
    pixels = pixels[order]
    key = key[order]
    batches, cur = [], []
    last = None
    for p, k in zip(pixels, key):
        if cur and (len(cur) >= batch or (k != last and len(cur) >= batch // 2)):
            batches.append(np.array(cur))
            cur = []
        cur.append(p)
        last = k
    if cur:
        batches.append(np.array(cur))
    return batches


def forward(scene, cam, model, background, *, max_splats=128, alpha_cutoff=1.0 / 255.0,
            near=1e-4, chunk_size=None, pixels=None, prune=True, batch=64,
            keep_state=False):
    """Forward sweep over ``pixels`` (flat indices; default all).

    Returns a dict of per-pixel arrays (rad (m,3), residual, overdraw, sat,
    e_k, t_k, theta0) in the order of ``pixels``; with ``keep_state`` also
    the per-batch replay state consumed by :func:`backward`.
    """
    scene = Scene.of(scene)
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    npx = cam.width * cam.height
    pixels = np.arange(npx) if pixels is None else np.asarray(pixels, dtype=np.int64)
    dirs_all = pixel_directions(cam)
    group, tie = _group_keys(scene, cam, chunk_size)
    keys = ("rad", "residual", "overdraw", "sat", "e_k", "t_k", "theta0", "amargin",
            "smargin", "tmargin")
    res = {k: None for k in keys}
    states = []
    pos = {int(p): i for i, p in enumerate(pixels)}
    for b in _pixel_batches(cam, pixels, batch):
        out, st = _forward_batch(scene, cam, model, bg, dirs_all[b], max_splats,
                                 alpha_cutoff, near, group, tie, prune)
        idx = np.array([pos[int(p)] for p in b])
        for k in keys:
            if res[k] is None:
                shp = (len(pixels),) + out[k].shape[1:]
                res[k] = np.zeros(shp, dtype=out[k].dtype)
            res[k][idx] = out[k]
        if keep_state:
            states.append((b, idx, out, st))
    if len(pixels) == 0:
        for k in keys:
            res[k] = np.zeros((0, 3) if k in ("rad", "e_k", "theta0") else (0,))
    res["pixels"] = pixels
    res["mask"] = margin_mask(res, model, t_order=(chunk_size != 1))
    if keep_state:
        res["_states"] = states
    return res


def margin_mask(res, model, tol=1e-5, t_order=False):
    """Pixels excluded from fp32-vs-fp64 parity because a decision sits on a
    threshold (the reference's own gradcheck excludes
    near-saturation rays the same way, adjoint.py:225-231).  True = masked."""
    m = res["amargin"] < tol
    if model.variant == "exponential":
        # the fp64 reference saturates exp only once T < ~1e-16; the fp32
        # device carries T = P and never does
        m = m | res["sat"]
    else:
        m = m | (res["smargin"] < tol)
    if t_order:  # candidates with |Δt| < 1e-6·t
        m = m | (res["tmargin"] < 1e-6)
    return m


# ---------------------------------------------------------------------------
# backward: unified adjoint (fp64, front-to-back) + parameter chain
# ---------------------------------------------------------------------------

def _backward_batch(scene, cam, model, bg, out, st, seed, grads, mass):
    variant, param = model.variant, float(getattr(model, "param", 0.0))
    slots = st["slots"]
    if not slots:
        return
    geo, Y, Epos = st["geo"], st["Y"], st["Epos"]
    ids = st["ids"]
    m = seed.shape[0]
    cols = np.arange(m)
    n_r = len(ids)
    e_k = out["e_k"]
    # per-slot adjoint quantities, (S, m)
    S = len(slots)
    go = np.stack([s[1] for s in slots])
    satn = np.stack([s[2] for s in slots])
    a = np.stack([s[3] for s in slots])
    E = np.stack([s[4] for s in slots])                       # (S, m, 3)
    tau_b = np.stack([s[5] for s in slots])
    prod_b = np.stack([s[6] for s in slots])
    w = np.stack([s[7] for s in slots])
    g, fp, gamma = weight_terms(variant, param, tau_b, prod_b)
    sdE = np.einsum("smc,mc->sm", E - e_k[None], seed)          # seed·(E_i - E_k)
    want_mag = mass is not None
    if want_mag:
        # absolute evaluation of the same sums (|terms| summed, Higham's
        # running-error scale): seed·(E_i - E_k) cancels, and so can the
        # adjoint d_alpha = sdE·g + Θ; an fp32 evaluation is accurate to
        # ~eps of these magnitudes, not of the cancelled result
        sdE_m = np.einsum("smc,mc->sm", np.abs(E) + np.abs(e_k[None]), np.abs(seed))
    if gamma == 0.0:
        # Θ_i = Σ_{j>i, go} sdE_j α_j f'(τ̄_j)
        term = np.where(go, sdE * a * fp, 0.0)
        suffix = np.cumsum(term[::-1], axis=0)[::-1] - term
        d_al = np.where(go, sdE * g + suffix, 0.0)
        if want_mag:
            tm = np.where(go, sdE_m * a * np.abs(fp), 0.0)
            sm = np.cumsum(tm[::-1], axis=0)[::-1] - tm
            d_al_m = np.where(go, sdE_m * np.abs(g) + sm, 0.0)
    else:
        # γ/(1-α_i) Σ_{j>i, go} sdE_j α_j P_j
        term = np.where(go, sdE * a * prod_b, 0.0)
        suffix = np.cumsum(term[::-1], axis=0)[::-1] - term
        d_al = np.where(go, sdE * g - gamma * suffix / (1.0 - a), 0.0)
        if want_mag:
            tm = np.where(go, sdE_m * a * np.abs(prod_b), 0.0)
            sm = np.cumsum(tm[::-1], axis=0)[::-1] - tm
            d_al_m = np.where(go, sdE_m * np.abs(g) + abs(gamma) * sm / (1.0 - a), 0.0)
    d_em = np.where(go[..., None], seed[None] * (a * g)[..., None], 0.0)
    d_em = np.where(satn[..., None], seed[None] * w[..., None], d_em)
    # scatter to (row, pixel)
    d_alpha_rows = np.zeros((n_r, m))
    d_em_rows = np.zeros((n_r, m, 3))
    d_alpha_m = np.zeros((n_r, m)) if want_mag else None
    for si, s in enumerate(slots):
        rows = s[0]
        d_alpha_rows[rows, cols] += d_al[si]
        d_em_rows[rows, cols] += d_em[si]
        if want_mag:
            d_alpha_m[rows, cols] += d_al_m[si]
    # chain, reference render.py:326-341
    d_alpha_rows = np.where(geo["clamped"], 0.0, d_alpha_rows)
    da = d_alpha_rows * geo["alpha"]
    u = np.einsum("rba,rmb->rma", geo["R"], geo["diff"])
    us2 = u / geo["s"][:, None, :] ** 2
    J = quat_rot_jacobian(geo["q"])
    dm2_dq = 2.0 * np.einsum("rqab,rma,rmb->rmq", J, geo["diff"], us2)
    qn = geo["q"]
    d_em_eff = np.where(Epos, d_em_rows, 0.0)

    t_op = d_alpha_rows * geo["kernel"]
    t_c = da[:, :, None] * geo["Adiff"]
    t_s = da[:, :, None] * (u * us2 / geo["s"][:, None, :])
    t_qu = (-0.5 * da)[:, :, None] * dm2_dq
    t_q = t_qu - qn[:, None, :] * np.einsum("rq,rmq->rm", qn, t_qu)[:, :, None]
    t_sh = np.einsum("rmc,mk->rmck", d_em_eff, Y)
    grads["opacities"][ids] += t_op.sum(1)
    grads["centers"][ids] += t_c.sum(1)
    grads["scales"][ids] += t_s.sum(1)
    grads["quats"][ids] += t_q.sum(1)
    grads["sh"][ids] += t_sh.sum(1)
    if mass is not None:
        # parity scale of each gradient entry: Σ over pixels of the term's
        # magnitude.  The geometric groups use the norm of the per-pixel
        # term VECTOR (normwise): a component that is small next to its
        # siblings (e.g. the thin-axis scale of a needle, or the ray-ward
        # centre component) is only defined to fp32 precision of the whole
        # per-pixel vector, which any fp32 evaluation of the peak offset
        # inherits
        mass["opacities"][ids] += np.abs(t_op).sum(1)
        mass["centers"][ids] += np.linalg.norm(t_c, axis=2).sum(1)[:, None]
        mass["scales"][ids] += np.linalg.norm(t_s, axis=2).sum(1)[:, None]
        mass["quats"][ids] += np.linalg.norm(t_q, axis=2).sum(1)[:, None]
        mass["sh"][ids] += np.abs(t_sh).sum(1)
        # componentwise scale (S = Σ_px |per-pixel term| of
        # that entry alone), each per-pixel term evaluated in absolute
        # values: |d_alpha| from its own terms (above), and |R|·|Λu| /
        # |J|·|diff|·|Λu| for the rotations that mix a term's components
        # (a centre component that is small next to its siblings is a
        # cancellation of the rotated offset, fp32-accurate only to ~eps of
        # the terms).  DESIGN.md §6 gives the measured cases that need it.
        d_alpha_m = np.where(geo["clamped"], 0.0, d_alpha_m)
        da_m = d_alpha_m * geo["alpha"]
        R_abs = np.abs(geo["R"])
        us2_abs = np.abs(us2)
        mass["opacities_c"][ids] += (d_alpha_m * geo["kernel"]).sum(1)
        mass["centers_c"][ids] += (da_m[:, :, None] * np.einsum("rab,rmb->rma", R_abs,
                                                                 us2_abs)).sum(1)
        mass["scales_c"][ids] += (da_m[:, :, None] * np.abs(u * us2 / geo["s"][:, None, :])).sum(1)
        tq_m = da_m[:, :, None] * np.einsum("rqab,rma,rmb->rmq", np.abs(J), np.abs(geo["diff"]),
                                            us2_abs)
        tq_m = tq_m + np.abs(qn)[:, None, :] * np.einsum("rq,rmq->rm", np.abs(qn), tq_m)[:, :, None]
        mass["quats_c"][ids] += tq_m.sum(1)
        mass["sh_c"][ids] += np.abs(t_sh).sum(1)


def _zero_grads(scene):
    P = len(scene)
    return {
        "centers": np.zeros((P, 3)),
        "scales": np.zeros((P, 3)),
        "quats": np.zeros((P, 4)),
        "opacities": np.zeros(P),
        "sh": np.zeros_like(scene.sh),
    }


def backward(scene, cam, model, background, fwd, seed, *, with_mass=False):
    """Gradients for ``seed`` (per-pixel d loss / d radiance, shape
    (len(pixels), 3) matching ``fwd['pixels']``, or (H, W, 3) for full
    images).  ``fwd`` must come from :func:`forward` with ``keep_state``."""
    scene = Scene.of(scene)
    bg = np.asarray(background, dtype=np.float64).reshape(3)
    seed = np.asarray(seed, dtype=np.float64).reshape(-1, 3)
    if seed.shape[0] == cam.width * cam.height and len(fwd["pixels"]) != seed.shape[0]:
        seed = seed[fwd["pixels"]]
    grads = _zero_grads(scene)
    mass = None
    if with_mass:
        mass = _zero_grads(scene)
        for k in ("centers", "scales", "quats", "opacities", "sh"):
            mass[k + "_c"] = np.zeros_like(mass[k])
    for b, idx, out, st in fwd["_states"]:
        _backward_batch(scene, cam, model, bg, out, st, seed[idx], grads, mass)
    if with_mass:
        return grads, mass
    return grads


def render_with_gradients(scene, cam, model, background, seed, *, with_mass=False, **kw):
    fwd = forward(scene, cam, model, background, keep_state=True, **kw)
    bw = backward(scene, cam, model, background, fwd, seed, with_mass=with_mass)
    return fwd, bw


# ---------------------------------------------------------------------------
# canonical synthetic scene and the fp32 protocol
# ---------------------------------------------------------------------------

def canonical_scene(n, seed=5, C=4):
    """A.1: generalises reference studies.py:170-181 (+142-143 SH draw)."""
    rng = np.random.default_rng(seed)
    s = (5000.0 / n) ** (1.0 / 3.0)
    centers = np.column_stack([rng.uniform(-1.6, 1.6, n), rng.uniform(-1.6, 1.6, n),
                               rng.uniform(2.0, 8.0, n)])
    scales = rng.uniform(0.05, 0.18, (n, 3)) * s
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opac = rng.uniform(0.3, 0.9, n)
    sh = np.zeros((n, 3, C))
    sh[:, :, 0] = rng.uniform(0.2, 1.0, (n, 3)) / SH_C0
    if C == 4:
        sh[:, :, 1:] = rng.normal(0.0, 0.15, (n, 3, 3))
    return Scene(centers, scales, quats, opac, sh)


def round_scene_f32(scene):
    """Parity protocol: every field -> float32 -> float64."""
    f = lambda x: np.asarray(x, dtype=np.float32).astype(np.float64)  # noqa: E731
    return Scene(f(scene.centers), f(scene.scales), f(scene.quats), f(scene.opacities),
                 f(scene.sh))


class _Cam:
    def __init__(self, position, rotation, focal, cx, cy, width, height):
        self.position = np.asarray(position, dtype=np.float64)
        self.rotation = np.asarray(rotation, dtype=np.float64)
        self.focal, self.cx, self.cy = float(focal), float(cx), float(cy)
        self.width, self.height = int(width), int(height)


def look_at(position, target, up, fov_deg, width, height):
    """reference primitives.py:172-190 (Camera.from_look_at)."""
    position = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd], axis=1)
    focal = 0.5 * width / np.tan(np.radians(fov_deg) / 2.0)
    return _Cam(position, R, focal, width / 2.0, height / 2.0, width, height)


def canonical_camera(width, height, view=0, n_views=1):
    """A.1/A.2 camera: view v of V at 0.4·(cos, sin)(2πv/V), looking at (0,0,3.5)."""
    if n_views <= 1:
        pos = [0.0, 0.0, 0.0]
    else:
        ang = 2.0 * np.pi * view / n_views
        pos = [0.4 * np.cos(ang), 0.4 * np.sin(ang), 0.0]
    return look_at(pos, [0.0, 0.0, 3.5], [0.0, 1.0, 0.0], 55.0, width, height)


def canonical_seed(width, height, view=0):
    """A.2 adjoint seed: U(0.2, 1) per channel from default_rng(1000+v)."""
    return np.random.default_rng(1000 + view).uniform(0.2, 1.0, (height, width, 3))

"""Data parallelism over camera views.

Views are independent units: every rank holds a full scene replica,
renders its share of the step's views (forward + backward, gradients
accumulating into ONE flat float32 buffer laid out as
[centers | scales | quats | opacities | sh]), then the ranks sum that
buffer with a single all-reduce (NCCL over NVLink/NVSwitch on B200,
``torch.distributed``).  The reference has no parallelism beyond row-band
threads in ``render`` (reference render.py:394-400); this layer is new.

The per-view work is pluggable (``render_view(view_index, grads)``), so
the host logic — view partition, flat-buffer layout, the all-reduce — is
tested on CPU with ``gloo`` and world size 2 (tests/test_dp.py).
"""
from __future__ import annotations

from dataclasses import dataclass

__all__ = ["partition_views", "GradBuffer", "DataParallelStep", "device_view_renderer",
           "sparse_allreduce"]


def partition_views(n_views: int, rank: int, world: int) -> list[int]:
    """Contiguous block partition of ``n_views`` over ``world`` ranks
    (⌈V/G⌉ per rank, the last ranks possibly fewer)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-n_views // world)
    lo = min(n_views, rank * per)
    return list(range(lo, min(n_views, lo + per)))


class GradBuffer:
    """One flat float32 buffer with per-field views shaped like the scene."""

    def __init__(self, n: int, sh_coeffs: int, device=None, dtype=None):
        import torch
        dtype = torch.float32 if dtype is None else dtype
        self.n, self.c = n, sh_coeffs
        self.sizes = {"centers": 3 * n, "scales": 3 * n, "quats": 4 * n, "opacities": n,
                      "sh": 3 * sh_coeffs * n}
        self.shapes = {"centers": (n, 3), "scales": (n, 3), "quats": (n, 4), "opacities": (n,),
                       "sh": (n, 3, sh_coeffs)}
        self.flat = torch.zeros(sum(self.sizes.values()), dtype=dtype, device=device)
        self.fields = {}
        off = 0
        for k, sz in self.sizes.items():
            self.fields[k] = self.flat[off:off + sz].view(self.shapes[k])
            off += sz

    def zero_(self):
        self.flat.zero_()

    def __getitem__(self, k):
        return self.fields[k]


def sparse_allreduce(grads: GradBuffer, group=None, dense_above: float = 0.5) -> int:
    """Sum the per-rank gradient buffers over the group, communicating only
    the Gaussians some rank touched.  A view touches the Gaussians of its
    processed depth phases (at C3 ~3% of the scene), so the all-reduce of
    the whole flat buffer moves mostly zeros.  Steps: an all-reduce (MAX) of
    the per-Gaussian "has a nonzero gradient" byte mask, then one all-reduce
    of the union's rows packed as (m, 23) and a scatter back.  Entries no
    rank touched are zero everywhere, so the result equals the dense sum
    (up to the order of the floating-point additions).  Falls back to the
    dense all-reduce when the union exceeds ``dense_above`` of the scene.
    Returns the number of Gaussians communicated."""
    import torch
    import torch.distributed as dist
    n = grads.n
    rows = {k: v.reshape(n, -1) for k, v in grads.fields.items()}
    mask = torch.zeros(n, dtype=torch.uint8, device=grads.flat.device)
    for t in rows.values():
        mask |= (t != 0).any(dim=1).to(torch.uint8)
    dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=group)
    idx = torch.nonzero(mask, as_tuple=False).squeeze(1)
    m = int(idx.numel())
    if m > dense_above * n:
        dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=group)
        return n
    if m == 0:
        return 0
    packed = torch.cat([t.index_select(0, idx) for t in rows.values()], dim=1)
    dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    off = 0
    for t in rows.values():
        w = t.shape[1]
        t.index_copy_(0, idx, packed[:, off:off + w])
        off += w
    return m


@dataclass
class DataParallelStep:
    """One data-parallel fwd+bwd step over ``n_views`` views: each rank
    renders its views into the flat gradient buffer, then the ranks sum it
    (``sparse``: only the Gaussians some rank touched, see
    :func:`sparse_allreduce`; else one all-reduce of the whole buffer)."""

    n_views: int
    rank: int
    world: int
    grads: GradBuffer
    render_view: object  # callable(view_index, grads: GradBuffer) -> None
    group: object = None
    sparse: bool = True

    def views(self) -> list[int]:
        return partition_views(self.n_views, self.rank, self.world)

    def __call__(self) -> GradBuffer:
        self.grads.zero_()
        for v in self.views():
            self.render_view(v, self.grads)
        if self.world > 1:
            if self.sparse:
                sparse_allreduce(self.grads, self.group)
            else:
                import torch.distributed as dist
                dist.all_reduce(self.grads.flat, op=dist.ReduceOp.SUM, group=self.group)
        return self.grads


def device_view_renderer(dev_scene, model, background, cameras, seeds, *, chunk_size=1,
                         max_splats=128, views=None, first_phase_ranks=0, deterministic=False):
    """Per-view fwd+bwd through libnxs on the current CUDA device.
    ``cameras[v]`` / ``seeds[v]`` (H,W,3 float32 CUDA) for view v; each view
    index gets its own persistent ``nxs_view`` workspace."""
    from . import _native
    from .render import forward_backward_device
    views = {} if views is None else views
    outs = {}

    def render_view(v, grads):
        if v not in views:
            views[v] = _native.View()
        # fused forward + backward; the output images are reused per view
        o, _ = forward_backward_device(views[v], dev_scene, cameras[v], model, background,
                                       seeds[v], grads.fields, chunk_size=chunk_size,
                                       max_splats=max_splats,
                                       first_phase_ranks=first_phase_ranks, out=outs.get(v),
                                       deterministic=deterministic)
        outs[v] = o

    render_view.views = views
    return render_view

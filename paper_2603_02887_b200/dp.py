"""Data parallelism over camera views.

Views are independent units: every rank holds a full scene replica,
renders its share of the step's views (forward + backward, gradients
accumulating into ONE flat float32 buffer laid out as
[centers | scales | quats | opacities | sh]), then the ranks sum that
buffer (NCCL over NVLink/NVSwitch on B200, ``torch.distributed``).  The
reference has no parallelism beyond row-band threads in ``render``
(reference render.py:394-400) and renders one view per optimizer iteration
(optimizer.py:393-408); this layer is new.

Touched rows.  A view's backward writes only the Gaussians of its processed
depth phases (~3 % of the scene at C3).  The library marks them in the
buffer's one-byte-per-Gaussian mask (``nxs_touched_mark``, no host sync);
the sparse reduction all-reduces that mask (MAX), selects the union
(``nxs_grads_select``: one host read of its size), gathers the union's rows
into one packed array, all-reduces it and scatters it back
(``nxs_grads_gather`` / ``_scatter``) — hand-written kernels, no eager
torch scans.  The mask then holds exactly the rows that are non-zero on
every rank, so the next step clears only those (``nxs_grads_zero_masked``)
instead of the whole 92 MB buffer.

Workspaces.  A rank keeps a small pool of ``nxs_view`` workspaces (about
0.7 GB each at C3, 3 GB at C5) and cycles its views through them; each
view's sizing history (first depth phase, pair count, key bins: a few
scalars, ``nxs_view_history_save/_load``) follows it from workspace to
workspace, so every view keeps the sync-free device-sized first phase.

The per-view work is pluggable (``render_view(view_index, grads)``); the
host logic is tested with ``gloo`` at world size 2 on CPU tensors
(tests/test_dp.py, a plain-torch restatement of the same reduction) and,
on a GPU, with two processes sharing it (tests/test_gpu_dp.py).
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
    """One flat float32 buffer with per-field views shaped like the scene,
    plus the per-Gaussian touched mask (uint8)."""

    def __init__(self, n: int, sh_coeffs: int, device=None, dtype=None):
        import torch
        dtype = torch.float32 if dtype is None else dtype
        self.n, self.c = n, sh_coeffs
        self.sizes = {"centers": 3 * n, "scales": 3 * n, "quats": 4 * n, "opacities": n,
                      "sh": 3 * sh_coeffs * n}
        self.shapes = {"centers": (n, 3), "scales": (n, 3), "quats": (n, 4), "opacities": (n,),
                       "sh": (n, 3, sh_coeffs)}
        self.flat = torch.zeros(sum(self.sizes.values()), dtype=dtype, device=device)
        self.mask = torch.zeros(n, dtype=torch.uint8, device=device)
        # True while `mask` flags every non-zero row: set by
        # device_view_renderer after it marks the rows a view wrote; any other
        # writer of the buffer must leave it False (the clear is then dense)
        self.mask_exact = False
        self.fields = {}
        off = 0
        for k, sz in self.sizes.items():
            self.fields[k] = self.flat[off:off + sz].view(self.shapes[k])
            off += sz

    @property
    def row_width(self) -> int:
        return 11 + 3 * self.c

    def zero_(self):
        """Clear the buffer: only the flagged rows when the mask is exact
        (the previous step's writes all went through a marking renderer)."""
        if self.flat.is_cuda and self.mask_exact and self.flat.dtype == torch_f32():
            from . import _native
            _native.grads_zero_masked(self.flat, self.n, self.c, self.mask)
        else:
            self.flat.zero_()
            self.mask.zero_()
        self.mask_exact = False

    def __getitem__(self, k):
        return self.fields[k]


def torch_f32():
    import torch
    return torch.float32


def _rows_cpu(grads: GradBuffer) -> dict:
    return {k: v.reshape(grads.n, -1) for k, v in grads.fields.items()}


def sparse_allreduce(grads: GradBuffer, group=None, dense_above: float = 0.5) -> int:
    """Sum the per-rank gradient buffers over the group, communicating only
    the Gaussians some rank touched: an all-reduce (MAX) of the touched
    mask, then one all-reduce of the union's rows packed (m, 11+3C) and a
    scatter back.  Rows no rank touched are zero everywhere, so the result
    equals the dense sum (up to the order of the floating-point additions).
    Falls back to the dense all-reduce when the union exceeds
    ``dense_above`` of the scene.  Returns the number of Gaussians
    communicated.  CUDA buffers use the library's kernels; CPU buffers (the
    gloo host-logic test) a plain-torch restatement."""
    import torch
    import torch.distributed as dist
    n = grads.n
    if not grads.flat.is_cuda:
        rows = _rows_cpu(grads)
        mask = torch.zeros(n, dtype=torch.uint8)
        for t in rows.values():
            mask |= (t != 0).any(dim=1).to(torch.uint8)
        grads.mask.copy_(mask)
    elif not grads.mask_exact:  # written by some other renderer: derive the mask
        grads.mask.zero_()
        for t in _rows_cpu(grads).values():
            grads.mask |= (t != 0).any(dim=1).to(torch.uint8)
        grads.mask_exact = True
    dist.all_reduce(grads.mask, op=dist.ReduceOp.MAX, group=group)
    if not grads.flat.is_cuda:
        idx = torch.nonzero(grads.mask, as_tuple=False).squeeze(1)
        m = int(idx.numel())
        if m > dense_above * n:
            dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=group)
            return n
        if m:
            packed = torch.cat([t.index_select(0, idx) for t in rows.values()], dim=1)
            dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
            off = 0
            for t in rows.values():
                w = t.shape[1]
                t.index_copy_(0, idx, packed[:, off:off + w])
                off += w
        return m
    from . import _native
    index = torch.empty(max(n, 1), dtype=torch.int32, device=grads.flat.device)
    m = _native.grads_select(grads.mask, n, index)
    if m > dense_above * n:
        dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=group)
        return n
    if m == 0:
        return 0
    packed = torch.empty((m, grads.row_width), dtype=torch.float32, device=grads.flat.device)
    _native.grads_gather(grads.flat, n, grads.c, index, m, packed)
    dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    _native.grads_scatter(grads.flat, n, grads.c, index, m, packed)
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
                if self.grads.flat.is_cuda and self.grads.mask_exact:
                    # rows touched on other ranks are now non-zero here too
                    dist.all_reduce(self.grads.mask, op=dist.ReduceOp.MAX, group=self.group)
        return self.grads


def device_view_renderer(dev_scene, model, background, cameras, seeds, *, chunk_size=1,
                         max_splats=128, pool=8, first_phase_ranks=0, deterministic=False):
    """Per-view fwd+bwd through libnxs on the current CUDA device.
    ``cameras[v]`` and ``seeds(v)`` (or ``seeds[v]``; H,W,3 float32 CUDA) for
    view v.  Views cycle through ``pool`` persistent ``nxs_view``
    workspaces (and output images); each marks the rows it wrote in the
    gradient buffer's mask."""
    from . import _native
    from .render import forward_backward_device
    workspaces: list = []
    outs: dict = {}
    history: dict = {}  # view index -> its sizing history (when views share workspaces)
    last_in: dict = {}  # workspace slot -> the view it served last
    pool = max(1, int(pool))

    def render_view(v, grads):
        slot = v % pool
        while len(workspaces) <= slot:
            workspaces.append(_native.View())
        view = workspaces[slot]
        prev = last_in.get(slot)
        if prev is not None and prev != v:  # the workspace changes camera
            history[prev] = view.history_save()
            if v in history:
                view.history_load(history[v])
        last_in[slot] = v
        seed = seeds(v) if callable(seeds) else seeds[v]
        # fused forward + backward; the output images are reused per slot
        o, _ = forward_backward_device(view, dev_scene, cameras[v], model, background, seed,
                                       grads.fields, chunk_size=chunk_size,
                                       max_splats=max_splats, first_phase_ranks=first_phase_ranks,
                                       out=outs.get(slot), deterministic=deterministic)
        outs[slot] = o
        view.touched_mark(grads.mask)
        grads.mask_exact = True  # (this step's earlier writes were marked too, or cleared)

    render_view.workspaces = workspaces
    render_view.outputs = outs
    return render_view

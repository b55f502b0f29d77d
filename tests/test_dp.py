"""Data parallelism over views: world size 2 with the gloo backend on CPU.

The per-view renderer is the CPU oracle here (the device renderer needs a
GPU); what is under test is the host logic of paper_2603_02887_b200.dp —
view partition, flat gradient buffer, the all-reduce — and that the
all-reduced buffer equals the sum of per-view reference gradients
(SURVEY §8e oracle)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_02887_b200.dp import DataParallelStep, GradBuffer, partition_views


def test_partition_covers_views_once():
    for V in (1, 5, 8, 64, 65):
        for G in (1, 2, 3, 4, 8):
            got = [v for r in range(G) for v in partition_views(V, r, G)]
            assert got == list(range(V))


def test_grad_buffer_layout():
    g = GradBuffer(5, 4)
    assert g.flat.numel() == 5 * (3 + 3 + 4 + 1 + 12)
    g["sh"][2, 1, 3] = 7.0
    off = 5 * (3 + 3 + 4 + 1) + (2 * 12 + 1 * 4 + 3)
    assert g.flat[off] == 7.0
    assert g["centers"].data_ptr() == g.flat.data_ptr()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from oracle import splat_oracle as O
    return O.round_scene_f32(O.canonical_scene(200, seed=3))


def _view_grads(v, n_views):
    from oracle import splat_oracle as O
    from tests._util import Model
    sc = _scene()
    cam = O.canonical_camera(24, 20, v, n_views)
    seed = O.canonical_seed(24, 20, v)
    _, g = O.render_with_gradients(sc, cam, Model("softplus", 20.0), np.zeros(3), seed,
                                   chunk_size=1)
    return g


def _worker(rank, world, port, n_views, out, sparse=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = _scene()
    grads = GradBuffer(len(sc), sc.sh.shape[2], dtype=torch.float64)

    def render_view(v, gb):
        g = _view_grads(v, n_views)
        for k, t in gb.fields.items():
            t += torch.from_numpy(np.ascontiguousarray(g[k]).reshape(t.shape))

    step = DataParallelStep(n_views, rank, world, grads, render_view, sparse=sparse)
    step()
    out[rank] = grads.flat.numpy().copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("sparse", [True, False])
@pytest.mark.parametrize("n_views", [2, 3])
def test_allreduce_equals_sum_of_per_view_gradients(n_views, sparse):
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, n_views, out, sparse), nprocs=world, join=True)
        res = dict(out)
    assert np.array_equal(res[0], res[1])
    sc = _scene()
    expect = GradBuffer(len(sc), sc.sh.shape[2], dtype=torch.float64)
    for v in range(n_views):
        g = _view_grads(v, n_views)
        for k, t in expect.fields.items():
            t += torch.from_numpy(np.ascontiguousarray(g[k]).reshape(t.shape))
    np.testing.assert_allclose(res[0], expect.flat.numpy(), rtol=1e-12, atol=1e-15)


def _sparse_worker(rank, world, port, out):
    """Disjoint and overlapping touched sets, and an all-zero rank."""
    from paper_2603_02887_b200.dp import sparse_allreduce
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = GradBuffer(10, 4, dtype=torch.float64)
    rng = np.random.default_rng(rank)
    rows = [1, 4, 7] if rank == 0 else [4, 5]
    for k, t in g.fields.items():
        r = t.reshape(10, -1)
        for i in rows:
            r[i] = torch.from_numpy(rng.normal(size=r.shape[1]))
    before = g.flat.clone()
    m = sparse_allreduce(g)
    out[rank] = (g.flat.numpy().copy(), before.numpy(), m)
    dist.destroy_process_group()


def test_sparse_allreduce_equals_dense_sum():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_sparse_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    total = res[0][1] + res[1][1]
    np.testing.assert_allclose(res[0][0], total, rtol=1e-15, atol=0)
    np.testing.assert_array_equal(res[0][0], res[1][0])
    assert res[0][2] == 4  # rows 1, 4, 5, 7

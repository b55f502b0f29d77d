"""The data-parallel device path with two processes sharing one
GPU: device_view_renderer + DataParallelStep, sparse (touched-row mask,
select / gather / all-reduce / scatter kernels) and dense, over gloo with
CUDA tensors, against the sum of the same views rendered in one process.
The step runs twice, so the second clear goes through the masked zero.
(One GPU only: the ranks' kernels never wait on each other; NCCL over
NVLink is exercised by the driver's multi-GPU bench.)"""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_VIEWS, W, H, P = 4, 320, 240, 200_000


def _setup():
    import torch
    from oracle import splat_oracle as O
    from paper_2603_02887_b200 import DeviceScene, TransmittanceModel
    sc = O.round_scene_f32(O.canonical_scene(P, seed=3))
    dev = DeviceScene.from_arrays(sc)
    cams = [O.canonical_camera(W, H, v, N_VIEWS) for v in range(N_VIEWS)]
    seeds = [torch.as_tensor(O.canonical_seed(W, H, v), dtype=torch.float32).cuda()
             for v in range(N_VIEWS)]
    return sc, dev, cams, seeds, TransmittanceModel.softplus(20.0)


def _worker(rank, world, port, out_dir, sparse, pool):
    import torch
    import torch.distributed as dist
    from paper_2603_02887_b200.dp import DataParallelStep, GradBuffer, device_view_renderer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, dev, cams, seeds, model = _setup()
    grads = GradBuffer(P, 4, device="cuda")
    rv = device_view_renderer(dev, model, np.zeros(3), cams, seeds, pool=pool)
    step = DataParallelStep(N_VIEWS, rank, world, grads, rv, sparse=sparse)
    for it in range(2):
        g = step()
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"r{rank}_it{it}.npy"), g.flat.cpu().numpy())
        np.save(os.path.join(out_dir, f"m{rank}_it{it}.npy"), g.mask.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _reference():
    """All views rendered in this process into one buffer (no collective)."""
    import torch
    from paper_2603_02887_b200.dp import DataParallelStep, GradBuffer, device_view_renderer
    sc, dev, cams, seeds, model = _setup()
    grads = GradBuffer(P, 4, device="cuda")
    rv = device_view_renderer(dev, model, np.zeros(3), cams, seeds, pool=N_VIEWS)
    g = DataParallelStep(N_VIEWS, 0, 1, grads, rv)()
    torch.cuda.synchronize()
    return g.flat.cpu().numpy(), g.mask.cpu().numpy()


@pytest.mark.parametrize("sparse,pool", [(True, 1), (False, 2)])
def test_two_ranks_sum_equals_single_process(sparse, pool):
    import torch.multiprocessing as mp
    ref, ref_mask = _reference()
    assert 0 < ref_mask.sum() < P // 2  # (the sparse path moves the union only)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d, sparse, pool), nprocs=2,
                           start_method="spawn")
        for rank in range(2):
            for it in range(2):
                got = np.load(os.path.join(d, f"r{rank}_it{it}.npy"))
                np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max(),
                                           err_msg=f"rank {rank} step {it}")
                mask = np.load(os.path.join(d, f"m{rank}_it{it}.npy"))
                # the mask flags every non-zero row (it drives the next clear)
                rows = np.zeros(P, bool)
                off = 0
                for w in (3, 3, 4, 1, 12):
                    rows |= (got[off:off + w * P].reshape(P, w) != 0).any(1)
                    off += w * P
                assert not (rows & (mask == 0)).any()


def test_masked_zero_select_gather_scatter_kernels():
    """The four dp kernels against plain torch on a random buffer."""
    import torch
    from paper_2603_02887_b200 import _native
    from paper_2603_02887_b200.dp import GradBuffer
    n = 10_000
    g = GradBuffer(n, 4, device="cuda")
    g.flat.normal_()
    mask = (torch.rand(n, device="cuda") < 0.1).to(torch.uint8)
    g.mask.copy_(mask)
    index = torch.empty(n, dtype=torch.int32, device="cuda")
    m = _native.grads_select(g.mask, n, index)
    ref_idx = torch.nonzero(mask).squeeze(1).to(torch.int32)
    assert m == ref_idx.numel() and torch.equal(index[:m], ref_idx)
    packed = torch.empty((m, 23), device="cuda")
    _native.grads_gather(g.flat, n, 4, index, m, packed)
    rows = torch.cat([v.reshape(n, -1) for v in g.fields.values()], 1)
    assert torch.equal(packed, rows[ref_idx.long()])
    before = g.flat.clone()
    _native.grads_scatter(g.flat, n, 4, index, m, packed * 2)
    rows2 = torch.cat([v.reshape(n, -1) for v in g.fields.values()], 1)
    assert torch.equal(rows2[ref_idx.long()], 2 * packed)
    keep = mask == 0
    rows0 = torch.cat([before[o:o + w * n].reshape(n, w) for o, w in
                       zip(np.cumsum([0, 3 * n, 3 * n, 4 * n, n]), (3, 3, 4, 1, 12))], 1)
    assert torch.equal(rows2[keep], rows0[keep])
    g.mask_exact = True  # (as device_view_renderer leaves it)
    g.zero_()
    rows3 = torch.cat([v.reshape(n, -1) for v in g.fields.values()], 1)
    assert (rows3[ref_idx.long()] == 0).all() and torch.equal(rows3[keep], rows0[keep])
    assert int(g.mask.sum()) == 0

"""CPU (gloo, world_size 2): host-side logic of the multi-GPU z-slab driver --
slab plans, batch-root rotation, broadcast data flow, per-voxel projection
order, slab gather. The compute hooks are an order-sensitive stub (no CUDA on
this box); the CUDA hooks are exercised by the GPU tests and bench.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1401_3615_b200 import distributed as D
from paper_1401_3615_b200 import synth
from paper_1401_3615_b200.geometry import VolumeGeometry

L, W, H, N, BATCH = 12, 7, 5, 11, 3


def stub_hooks():
    nb = W * H * 4

    def pack(raw, packed, err):
        n = raw.shape[0]
        packed[: n * nb].copy_(raw.reshape(-1).view(torch.uint8))

    def back(vol, z0, z1, packed, n, mats, err):
        imgs = packed[: n * nb].view(torch.float32).reshape(n, H, W)
        z = torch.arange(z0, z1, dtype=torch.float32).reshape(-1, 1, 1)
        for j in range(n):
            # order-sensitive update: acc = 0.5*acc + f(projection, z, matrix)
            f = imgs[j].sum() * (z + 1.0) + float(mats[j][0])
            vol.mul_(0.5).add_(f)

    return D.Hooks(pack, back, nb)


def sequential_reference(imgs, mats):
    vol = torch.zeros((L, L, L))
    z = torch.arange(0, L, dtype=torch.float32).reshape(-1, 1, 1)
    for j in range(N):
        vol.mul_(0.5).add_(torch.from_numpy(imgs[j]).sum() * (z + 1.0) + float(mats[j][0]))
    return vol.numpy()


def data():
    r = np.random.default_rng(5)
    imgs = r.standard_normal((N, H, W)).astype(np.float32)
    mats = r.standard_normal((N, 12))
    return imgs, mats


def worker(rank, world, port, slabs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        imgs, mats = data()
        # each rank only holds the batches it uploads; the rest is garbage
        mine = np.full_like(imgs, np.nan)
        for first, n, root in D.batch_roots(N, BATCH, world):
            if root == rank:
                mine[first:first + n] = imgs[first:first + n]
        rec = D.DistributedReconstructor(VolumeGeometry.centered(L, 1.0), W, H, batch=BATCH,
                                         slabs=slabs, device="cpu", hooks=stub_hooks())
        slab = rec.reconstruct(torch.from_numpy(mine), mats)
        full = rec.gather(slab)
        if rank == 0:
            q.put(full)
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("slabs", [None, [(0, 3), (3, L)]])
def test_two_ranks_match_sequential(slabs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, slabs, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    imgs, mats = data()
    ref = sequential_reference(imgs, mats)
    assert np.array_equal(full, ref)


def test_slab_plans():
    assert D.equal_slabs(10, 3) == [(0, 3), (3, 6), (6, 10)]
    roots = D.batch_roots(100, 32, 3)
    assert [r for _, _, r in roots] == [0, 1, 2, 0]
    assert sum(n for _, n, _ in roots) == 100
    cfg = synth.CONFIGS[2]
    mats = synth.perturbed_matrices(cfg)
    g = cfg.geometry
    work = D.plane_work(g, mats[::8], cfg.width, cfg.height)
    assert work.shape == (512,)
    # centre planes see the detector from every angle, the top/bottom less
    assert work[256] > work[0] and work[256] > work[511]
    for world in (2, 4, 8):
        sl = D.balanced_slabs(work, world)
        assert sl[0][0] == 0 and sl[-1][1] == 512
        assert all(a < b for a, b in sl) and all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
        per = [work[a:b].sum() for a, b in sl]
        assert max(per) / (sum(per) / world) < 1.05
        eq = [work[a:b].sum() for a, b in D.equal_slabs(512, world)]
        assert max(per) <= max(eq)


def error_worker(rank, world, port, q):
    """Rank 1's slab flags w == 0 in one batch; rank 0 flags nothing. Both
    ranks must raise the same error (flags are OR-reduced over the group), and
    the uploading rank alone scans each batch (Hooks.check)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        imgs, mats = data()
        base = stub_hooks()
        checked = []

        def back(vol, z0, z1, packed, n, m, err):
            base.backproject(vol, z0, z1, packed, n, m, err)
            if z0 > 0 and np.any(np.asarray(m)[:, 0] == mats[4][0]):
                err |= 1

        def check(raw, err):
            checked.append(int(raw.shape[0]))

        hooks = D.Hooks(base.pack, back, base.packed_bytes, check)
        rec = D.DistributedReconstructor(VolumeGeometry.centered(L, 1.0), W, H, batch=BATCH,
                                         device="cpu", hooks=hooks)
        try:
            rec.reconstruct(torch.from_numpy(imgs), mats)
            q.put((rank, "no error", checked))
        except Exception as e:  # noqa: BLE001
            q.put((rank, type(e).__name__, checked))
    finally:
        dist.destroy_process_group()


def test_errors_reach_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=error_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[1] for o in out] == ["GeometryError", "GeometryError"]
    # batches of 3 over 11 projections: roots 0, 1, 0, 1 -> sizes (3, 3) / (3, 2)
    assert out[0][2] == [3, 3] and out[1][2] == [3, 2]


def test_rebalance_slabs_from_measured_times():
    """A cost the estimate gets wrong (outer planes 1.6x dearer than
    estimated): rebalancing from the measured per-slab times brings the
    max/mean imbalance from up to 1.35 to < 1.06 in one round and < 1.03 in
    two."""
    L = 512
    z = np.arange(L)
    est = 1.0 + np.exp(-((z - 256) / 150.0) ** 2)           # estimated work
    true = est * np.where(np.abs(z - 256) > 150, 1.6, 1.0)  # real cost
    for world in (2, 4, 8):
        sl = D.balanced_slabs(est, world)
        t = [true[a:b].sum() for a, b in sl]
        imb0 = max(t) / np.mean(t)
        sl2 = D.rebalance_slabs(est, sl, t)
        assert sl2[0][0] == 0 and sl2[-1][1] == L
        assert all(sl2[i][1] == sl2[i + 1][0] for i in range(world - 1))
        t2 = [true[a:b].sum() for a, b in sl2]
        imb1 = max(t2) / np.mean(t2)
        sl3 = D.rebalance_slabs(est, sl2, t2)
        t3 = [true[a:b].sum() for a, b in sl3]
        imb2 = max(t3) / np.mean(t3)
        assert imb1 < 1.06 and imb2 < 1.03, (world, imb0, imb1, imb2)
        assert world == 2 or imb0 > 1.15

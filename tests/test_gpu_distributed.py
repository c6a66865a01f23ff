"""The torch.distributed z-slab driver with the CUDA hooks at world size 2,
both ranks on the one GPU of the test box and the gloo backend standing in
for NCCL (host-level collectives only; no kernel waits on another rank):
rotating upload roots, broadcast, per-slab row bands, uploading-rank
validation, OR-reduced error flags -- the slabs, assembled here, bitwise
against the oracle. (gather() is not used: gloo has no CUDA send/recv.) A
functional check of the multi-process logic, not a measurement."""
import os
import socket

import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scan(kind):
    """(cfg, geometry, mats, imgs on the CPU): 'coarse' = config 0's scan into
    64^3 (gather kernel), 'staged' = config 2's scan into a central 96^3
    sub-cube at 0.5 mm (TMA-staged raw kernel)."""
    from paper_1401_3615_b200 import synth
    from paper_1401_3615_b200.geometry import VolumeGeometry

    if kind == "coarse":
        cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=64, num_projections=40)
        g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=20)
        return cfg, g, mats, imgs
    cfg = synth.CONFIGS[2]
    _, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=20, count=40)
    return cfg, VolumeGeometry.centered(96, cfg.voxel_mm), mats, imgs


def _worker(rank, world, port, q, transport="nccl", kind="coarse"):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1401_3615_b200.distributed import DistributedReconstructor, balanced_slabs, plane_work

        cfg, g, mats, imgs = _scan(kind)
        slabs = balanced_slabs(plane_work(g, mats, cfg.width, cfg.height), world)
        rec = DistributedReconstructor(g, cfg.width, cfg.height, batch=6, slabs=slabs,
                                       transport=transport)
        slab = rec.reconstruct(imgs.pin_memory(), mats)
        bad = imgs.clone()
        bad[13, 0, 0] = float("nan")  # batch 2 -> uploaded by rank 0
        try:
            rec.reconstruct(bad.pin_memory(), mats)
            err = "none"
        except Exception as e:  # noqa: BLE001
            err = type(e).__name__
        again = rec.reconstruct(imgs.pin_memory(), mats)  # flags keep counting
        rec.close()
        q.put((rank, np.array(slab), err, slabs, bool(np.array_equal(again, slab))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport,kind", [("nccl", "coarse"), ("ipc", "coarse"),
                                            ("nccl", "staged"), ("ipc", "staged")])
def test_two_rank_driver_on_one_gpu(cuda, oracle, transport, kind):
    """transport 'nccl': broadcast of each batch (gloo stands in here);
    transport 'ipc': every rank's pack reads the uploading rank's slot through
    CUDA IPC, ordered by stream flags (same device here, NVLink peers on a
    multi-GPU box)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, transport, kind))
             for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=180) for _ in range(2)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg, g, mats, imgs = _scan(kind)
    L = g.edge_voxels
    ref = np.zeros((L,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs.numpy(), mats) == 0
    slabs = out[0][3]
    assert slabs[0] == (0, slabs[0][1]) and slabs[0][1] == slabs[1][0] and slabs[1][1] == L
    full = np.concatenate([out[0][1], out[1][1]])
    assert bits_equal(full, ref)
    assert [o[2] for o in out] == ["ValidationError", "ValidationError"]
    assert all(o[4] for o in out)  # a second call on the same driver, same bits

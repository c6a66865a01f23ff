"""Seeded fuzz of the whole host pipeline against the oracle (bitwise):
random circular scans (source distance, magnification, detector size and
pitch, angular range, volume size and voxel size, volume offset from the
isocentre so the detector is over- or under-filled), random batch sizes,
1-4 slab workers sharing the GPU (rotating upload roots, row bands, peer band
copies), resident tail on or off, random initial volumes with -0.0 voxels,
contiguous / per-image / pageable / file / session inputs. A few cases use random
matrices (w changes sign -> guarded kernel, possibly w == 0 -> GeometryError
with the volume untouched)."""
import math
import os

import numpy as np
import pytest

from conftest import bits_equal

import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200.geometry import (TrajectoryConfig, VolumeGeometry,
                                           make_circular_trajectory)

pytestmark = pytest.mark.gpu


def case(seed):
    r = np.random.default_rng(seed)
    L = int(r.integers(12, 49)) if seed % 8 else int(r.integers(64, 97))  # some resident-size slabs
    W = int(r.integers(6, 90))
    H = int(r.integers(6, 70))
    n = int(r.integers(1, 45))
    voxel = float(r.uniform(0.3, 3.0))
    sid = float(r.uniform(60.0, 400.0))
    sdd = sid * float(r.uniform(1.1, 2.5))
    # pixel pitch so that the detector covers 40 %-160 % of the volume
    cover = float(r.uniform(0.4, 1.6))
    pitch = cover * L * voxel * (sdd / sid) / max(W, H)
    rng_deg = float(r.choice([180.0, 200.0, 360.0]))
    cfg = TrajectoryConfig(n, sid, sdd, W, H, pitch, math.radians(rng_deg))
    mats = make_circular_trajectory(cfg)
    if seed % 7 == 3:  # random matrices: w changes sign over the volume
        mats = r.standard_normal((n, 12))
        mats[:, 11] += 2.0
    origin = -0.5 * (L - 1) * voxel + float(r.uniform(-0.3, 0.3)) * L * voxel
    g = VolumeGeometry(L, voxel, origin)
    imgs = r.standard_normal((n, H, W)).astype(np.float32)
    imgs[r.random((n, H, W)) < 0.2] = 0.0
    vol0 = (r.standard_normal((L, L, L)) * float(r.choice([0.0, 1.0]))).astype(np.float32)
    if r.random() < 0.3:
        vol0[r.random(vol0.shape) < 0.1] = -0.0
    k = int(r.integers(1, 5))
    opts = dict(batch=int(r.integers(1, 33)), device_ids=[0] * k,
                mode=pkg.MODE_EXACT, cull=bool(r.random() < 0.85))
    return g, mats, imgs, vol0, opts, r


@pytest.mark.parametrize("seed", range(int(os.environ.get("CBB_FUZZ_SEEDS", "96"))))
def test_fuzz_pipeline_vs_oracle(cuda, oracle, monkeypatch, tmp_path, seed):
    g, mats, imgs, vol0, opts, r = case(seed)
    ref = vol0.copy()
    status = oracle.reconstruct(ref, g, imgs, mats)
    if r.random() < 0.5:
        monkeypatch.setenv("CBB_NO_RESIDENT", "1")
    how = ["contiguous", "images", "pageable", "file", "session"][seed % 5]
    v = vol0.copy()

    def run():
        if how == "contiguous":
            vol = pkg.Volume(g, v)
            return pkg.reconstruct(vol, pkg.ProjectionStack(g, mats, imgs), pkg.Options(**opts))
        if how == "images":
            return pkg.reconstruct_images(v, g, [np.array(a) for a in imgs], mats,
                                          pkg.Options(**opts))
        if how == "pageable":
            return pkg.reconstruct_arrays(v, g, np.array(imgs), mats, pkg.Options(**opts))
        if how == "session":  # per-projection calls, flushed in batches
            with pkg.Session(g, imgs.shape[2], imgs.shape[1], v, pkg.Options(**opts)) as sess:
                for i in range(len(mats)):
                    sess.backproject(imgs[i], mats[i])
                out, st = sess.finish()
            v[...] = out
            return st
        p = str(tmp_path / f"s{seed}.cbps")
        pkg.write_stack(p, pkg.ProjectionStack(g, mats, imgs))
        out, st = pkg.reconstruct_file(p, pkg.Options(**opts), initial=pkg.Volume(g, v))
        v[...] = out.voxels
        return st

    if status != 0:
        assert status == 5
        with pytest.raises(pkg.GeometryError):
            run()
        assert bits_equal(v, vol0)
        return
    run()
    assert bits_equal(v, ref), (seed, how, opts)
    if seed % 3 == 0 and seed % 7 != 3:  # fast mode within north_star's tolerance
        fast = pkg.Volume(g, vol0.copy())
        pkg.reconstruct(fast, pkg.ProjectionStack(g, mats, imgs),
                        pkg.Options(**dict(opts, mode=pkg.MODE_FAST)))
        d = fast.voxels.astype(np.float64) - ref
        rng = float(ref.max() - ref.min()) or 1.0
        assert np.linalg.norm(d) <= 1e-5 * max(np.linalg.norm(ref.astype(np.float64)), 1e-30)
        assert np.abs(d).max() <= 1e-4 * rng


def raw_case(seed):
    """Scans whose one-GPU reconstruction takes the TMA-staged raw mode: rows
    16-byte aligned (W % 4 == 0) and detector pixels fine enough relative to
    the voxels that the footprint boxes fit the staging budget."""
    r = np.random.default_rng(10_000 + seed)
    L = int(r.integers(16, 80))
    cover = float(r.uniform(0.5, 1.5))
    px = float(r.uniform(1.0, 3.2))  # detector pixels per voxel (at the isocentre)
    W = max(8, 4 * int(round(px * L * cover / 4)))
    H = max(6, int(W * float(r.uniform(0.4, 1.0))))
    n = int(r.integers(1, 70))
    voxel = float(r.uniform(0.3, 3.0))
    sid = float(r.uniform(60.0, 400.0))
    sdd = sid * float(r.uniform(1.1, 2.5))
    pitch = cover * L * voxel * (sdd / sid) / W
    rng_deg = float(r.choice([180.0, 200.0, 360.0]))
    mats = make_circular_trajectory(TrajectoryConfig(n, sid, sdd, W, H, pitch,
                                                     math.radians(rng_deg)))
    origin = -0.5 * (L - 1) * voxel + float(r.uniform(-0.3, 0.3)) * L * voxel
    g = VolumeGeometry(L, voxel, origin)
    imgs = r.standard_normal((n, H, W)).astype(np.float32)
    imgs[r.random((n, H, W)) < 0.2] = 0.0
    vol0 = (r.standard_normal((L, L, L)) * float(r.choice([0.0, 1.0]))).astype(np.float32)
    if r.random() < 0.3:
        vol0[r.random(vol0.shape) < 0.1] = -0.0
    k = int(r.choice([1, 1, 2, 3]))  # slab workers on the one GPU
    opts = dict(batch=int(r.integers(1, 65)), device_ids=[0] * k, cull=bool(r.random() < 0.85),
                ramp_filter_pixel_mm=None)
    return g, mats, imgs, vol0, opts, r


@pytest.mark.parametrize("seed", range(int(os.environ.get("CBB_FUZZ_RAW_SEEDS", "48"))))
def test_fuzz_raw_mode_vs_oracle(cuda, oracle, monkeypatch, seed):
    """The staged (raw-mode) pipeline on random scans, bitwise against the
    oracle: 1-3 slab workers (band rows copied from the uploading worker),
    upload batches 1-64, resident tail on/off, forced small boxes
    (global-memory taps) in a third of the cases, contiguous / per-image /
    pageable inputs."""
    g, mats, imgs, vol0, opts, r = raw_case(seed)
    n, H, W = imgs.shape
    if r.random() < 0.33:
        monkeypatch.setenv("CBB_TMA_BOX", "48x12")
    if r.random() < 0.5:
        monkeypatch.setenv("CBB_NO_RESIDENT", "1")
    staged = pkg.tma_plan(g, W, H, 0, g.edge_voxels, mats)["staged"]
    ref = vol0.copy()
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    v = vol0.copy()
    o = pkg.Options(**{k: val for k, val in opts.items() if val is not None})
    how = ["contiguous", "images", "pageable"][seed % 3]
    if how == "contiguous":
        vol = pkg.Volume(g, v)
        pkg.reconstruct(vol, pkg.ProjectionStack(g, mats, imgs), o)
        v = vol.voxels
    elif how == "images":
        pkg.reconstruct_images(v, g, [np.array(a) for a in imgs], mats, o)
    else:
        pkg.reconstruct_arrays(v, g, np.array(imgs), mats, o)
    assert bits_equal(v, ref), (seed, how, opts, staged)


def test_fuzz_raw_mode_mostly_staged():
    """Most raw_case scans really take the staged path (host-side plan)."""
    staged = 0
    for seed in range(48):
        g, mats, imgs, *_ = raw_case(seed)
        n, H, W = imgs.shape
        staged += pkg.tma_plan(g, W, H, 0, g.edge_voxels, mats)["staged"]
    assert staged >= 24, staged

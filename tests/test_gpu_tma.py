"""GPU: the TMA-staged back-projection from raw projections (bp_tma.cuh) --
bitwise against the oracle and against the packed-quad kernel, through the
device entry points (cbb_scan_device + cbb_backproject_raw_device) and the
single-GPU pipeline's raw mode (cbb_reconstruct), including its slow paths:
blocks whose footprint overflows the staged box (global-memory taps),
guarded batches, the IEEE-division redo for extreme numerators, row bands,
-0.0 voxels and culling statistics.

Geometry: BASELINE config 2's scan (1248 x 960 detector at 0.32 mm, 200 deg)
with a central 96^3 sub-cube at config 2's 0.5 mm voxels, so the footprint
boxes are the headline configuration's while the oracle stays fast.
"""
import numpy as np
import pytest

from conftest import bits_equal

import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200 import synth
from paper_1401_3615_b200.geometry import VolumeGeometry

pytestmark = pytest.mark.gpu

L = 96


@pytest.fixture(scope="module")
def scan(cuda):
    cfg = synth.CONFIGS[2]
    _, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=20, count=40)
    g = VolumeGeometry.centered(L, cfg.voxel_mm)
    return g, mats, imgs


@pytest.fixture(scope="module")
def expected(scan, oracle):
    g, mats, imgs = scan
    ref = np.zeros((L, L, L), np.float32)
    assert oracle.reconstruct(ref, g, imgs.cpu().numpy(), mats) == 0
    return ref


def raw_device(g, mats, imgs, vol0=None, z=(0, L), band=None, **opt):
    import torch

    n, H, W = imgs.shape
    flags = torch.zeros(n, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    src = imgs if band is None else imgs[:, band.raw_row0:band.raw_row0 + band.raw_rows].contiguous()
    pkg.scan_device(src, flags, err)
    v = torch.zeros((z[1] - z[0], L, L), dtype=torch.float32, device="cuda")
    if vol0 is not None:
        v.copy_(torch.from_numpy(vol0[z[0]:z[1]]))
    pkg.backproject_raw_device(v, g, z[0], z[1], src, W, H, n, mats, flags, pkg.Options(**opt),
                               err, band=band)
    torch.cuda.synchronize()
    return v.cpu().numpy(), int(err.item())


def test_plan_stages_this_geometry(scan):
    g, mats, imgs = scan
    n, H, W = imgs.shape
    p = pkg.tma_plan(g, W, H, 0, L, mats)
    assert p["staged"] == 1 and p["box_width"] >= p["footprint_width"]


def test_raw_device_path_bitwise(scan, expected):
    g, mats, imgs = scan
    v, err = raw_device(g, mats, imgs)
    assert err == 0
    assert bits_equal(v, expected)
    # uneven slab split: each slab is its own launch grid
    parts = [raw_device(g, mats, imgs, z=z)[0] for z in ((0, 37), (37, 61), (61, L))]
    assert bits_equal(np.concatenate(parts), expected)


def test_raw_path_equals_quad_path_fast_mode(scan):
    import torch

    g, mats, imgs = scan
    n, H, W = imgs.shape
    v, _ = raw_device(g, mats, imgs, mode=pkg.MODE_FAST)
    nb = pkg.packed_layout(W, H)[2]
    packed = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
    pkg.pack_device(imgs, packed)
    vq = torch.zeros((L, L, L), dtype=torch.float32, device="cuda")
    pkg.backproject_device(vq, g, 0, L, packed, W, H, n, mats, pkg.Options(mode=pkg.MODE_FAST))
    assert bits_equal(v, vq.cpu().numpy())


def test_overflowing_boxes_read_global_taps(scan, expected, monkeypatch):
    """A forced 48 x 12 box is smaller than most blocks' footprints: those
    (block, projection) pairs read their taps from global memory with the
    reference's bounds checks -- same bits."""
    g, mats, imgs = scan
    monkeypatch.setenv("CBB_TMA_BOX", "48x12")
    n, H, W = imgs.shape
    assert pkg.tma_plan(g, W, H, 0, L, mats)["box_rows"] == 12
    v, err = raw_device(g, mats, imgs)
    assert err == 0 and bits_equal(v, expected)


def test_guarded_raw_kernel(scan, expected, monkeypatch):
    g, mats, imgs = scan
    monkeypatch.setenv("CBB_FORCE_GUARDED", "1")
    v, err = raw_device(g, mats, imgs)
    assert err == 0 and bits_equal(v, expected)


def test_w_zero_flags_geometry_error(scan):
    g, mats, imgs = scan
    bad = mats.copy()
    bad[3] = 0.0
    bad[3, 0] = bad[3, 4] = 1.0  # w == 0 everywhere for projection 3
    v, err = raw_device(g, bad, imgs)
    assert err & 1


@pytest.mark.parametrize("scale_exp", [105, 90, -75])
def test_extreme_numerators_take_the_ieee_redo(scan, oracle, scale_exp):
    """Pixels >= 2^86 (flagged by the scan) or tiny nonzero numerators
    (tracked per voxel) make the thread redo the batch with IEEE divisions
    from the raw projections: bitwise the reference."""
    g, mats, imgs = scan
    h = imgs.cpu().numpy().astype(np.float64)
    h[5] *= 2.0 ** scale_exp
    h[17] *= 2.0 ** scale_exp
    h = h.astype(np.float32)
    ref = np.zeros((L, L, L), np.float32)
    assert oracle.reconstruct(ref, g, h, mats) == 0
    import torch

    v, err = raw_device(g, mats, torch.from_numpy(h).cuda())
    assert err == 0 and bits_equal(v, ref)


def test_row_band_buffers(scan, expected):
    """Slab workers holding only their row band (raw rows [r0, r0 + rn)):
    the tensor map covers the band, rows outside it read as zero."""
    g, mats, imgs = scan
    n, H, W = imgs.shape
    parts = []
    for z in ((0, 48), (48, L)):
        band = pkg.row_band_for_slab(g, W, H, z[0], z[1], mats)
        assert band.raw_rows < H
        parts.append(raw_device(g, mats, imgs, z=z, band=band)[0])
    assert bits_equal(np.concatenate(parts), expected)


def test_negative_zero_voxels_and_culling(scan, oracle):
    """-0.0 voxels switch culling off for their warp (-0 + +0 = +0); an
    initial volume of -0.0 with a few nonzero voxels, culling on and off."""
    g, mats, imgs = scan
    vol0 = np.full((L, L, L), -0.0, np.float32)
    vol0[::7, ::5, ::3] = 1.5
    ref = vol0.copy()
    assert oracle.reconstruct(ref, g, imgs.cpu().numpy(), mats) == 0
    for cull in (True, False):
        v, err = raw_device(g, mats, imgs, vol0=vol0, cull=cull)
        assert err == 0 and bits_equal(v, ref)


def test_negative_zero_voxels_off_centre(scan, oracle):
    """-0.0 voxels where culling does skip work (an off-centre cube past the
    detector edge): exact mode recomputes their threads with IEEE divisions
    (bitwise the oracle); fast mode switches culling off for their warps
    (culling on = culling off, bitwise)."""
    g0, mats, imgs = scan
    g = VolumeGeometry(L, g0.voxel_mm, 60.0)
    host = imgs.cpu().numpy()
    n, H, W = host.shape
    assert pkg.tma_plan(g, W, H, 0, L, mats)["staged"] == 1
    r = np.random.default_rng(7)
    vol0 = np.zeros((L, L, L), np.float32)
    vol0[r.random(vol0.shape) < 0.05] = -0.0
    vol0[:, :8, :] = -0.0
    vol0[::9, ::4, ::5] = 0.25
    ref = vol0.copy()
    assert oracle.reconstruct(ref, g, host, mats) == 0
    v, err = raw_device(g, mats, imgs, vol0=vol0)
    assert err == 0 and bits_equal(v, ref)
    fast = [raw_device(g, mats, imgs, vol0=vol0, mode=pkg.MODE_FAST, cull=c)[0]
            for c in (True, False)]
    assert bits_equal(fast[0], fast[1])


@pytest.mark.parametrize("resident", [True, False])
def test_pipeline_raw_mode(scan, expected, monkeypatch, resident):
    """cbb_reconstruct on one GPU with the whole stack known runs in raw mode
    (scan + TMA kernel, resident raw stack and tail, or a ring of raw slots);
    counting statistics equal the quad path's."""
    g, mats, imgs = scan
    if not resident:
        monkeypatch.setenv("CBB_NO_RESIDENT", "1")
    host = imgs.cpu().numpy()
    v = np.zeros((L, L, L), np.float32)
    st = pkg.reconstruct_arrays(v, g, host, mats, pkg.Options(num_gpus=1, batch=8,
                                                                count_culled=True))
    assert bits_equal(v, expected) and st["guarded_batches"] == 0
    monkeypatch.setenv("CBB_BP_PATH", "quad")
    vq = np.zeros((L, L, L), np.float32)
    stq = pkg.reconstruct_arrays(vq, g, host, mats, pkg.Options(num_gpus=1, batch=8,
                                                                  count_culled=True))
    assert bits_equal(vq, expected)
    # both count only provably-zero (culled) updates; the TMA kernel's warp
    # tiles differ from the quad kernel's, so the fractions are close, not equal
    assert abs(st["culled_fraction"] - stq["culled_fraction"]) < 0.1


def test_pipeline_raw_mode_off_centre_culling(scan, oracle):
    """An off-centre sub-cube reaching past the detector edge: culling skips
    part of the work (counted), results stay bitwise."""
    g0, mats, imgs = scan
    g = VolumeGeometry(L, g0.voxel_mm, 60.0)  # x, y, z from 60 mm to 107.5 mm
    host = imgs.cpu().numpy()
    ref = np.zeros((L, L, L), np.float32)
    assert oracle.reconstruct(ref, g, host, mats) == 0
    n, H, W = host.shape
    assert pkg.tma_plan(g, W, H, 0, L, mats)["staged"] == 1
    v = np.zeros((L, L, L), np.float32)
    st = pkg.reconstruct_arrays(v, g, host, mats, pkg.Options(num_gpus=1, count_culled=True))
    assert bits_equal(v, ref)
    assert st["culled_fraction"] > 0.01


def test_pipeline_raw_mode_filter_and_nan(scan, oracle, monkeypatch):
    """Raw mode with the GPU ramp filter (in place on the raw slots) equals
    back-projecting the device-filtered data; a NaN pixel is rejected."""
    import torch

    g, mats, imgs = scan
    cfg = synth.CONFIGS[2]
    raw = imgs.clone()
    filt = torch.empty_like(raw)
    pkg.ramp_filter_device(raw, filt, cfg.pixel_mm)
    ref = np.zeros((L, L, L), np.float32)
    assert oracle.reconstruct(ref, g, filt.cpu().numpy(), mats) == 0
    v = np.zeros((L, L, L), np.float32)
    pkg.reconstruct_arrays(v, g, raw.cpu().numpy(), mats,
                           pkg.Options(num_gpus=1, ramp_filter_pixel_mm=cfg.pixel_mm))
    assert bits_equal(v, ref)
    bad = imgs.cpu().numpy().copy()
    bad[11, 400, 600] = np.nan
    v = np.zeros((L, L, L), np.float32)
    with pytest.raises(pkg.ValidationError, match="ProjectionImage contains non-finite"):
        pkg.reconstruct_arrays(v, g, bad, mats, pkg.Options(num_gpus=1))
    assert not v.any()


@pytest.mark.parametrize("tail", [None, "12:36", "36:60"])
def test_pipeline_raw_mode_guarded_batch_with_resident_tail(scan, oracle, monkeypatch, tail):
    """A matrix with a -0.0 coefficient sends its batch to the guarded kernel
    (bp_guarded_raw); in raw mode with the resident tail its head launch must
    skip exactly the tail planes the staged kernel skips (same z-blocks, also
    for tails that do not start at a multiple of 8 planes)."""
    g, mats, imgs = scan
    if tail:
        monkeypatch.setenv("CBB_TAIL_PLANES", tail)
    m = mats.copy()
    m[9, 8] = -0.0  # a8 = -0: w no longer depends on z for projection 9
    host = imgs.cpu().numpy()
    ref = np.zeros((L, L, L), np.float32)
    assert oracle.reconstruct(ref, g, host, m) == 0
    v = np.zeros((L, L, L), np.float32)
    st = pkg.reconstruct_arrays(v, g, host, m, pkg.Options(num_gpus=1, batch=8))
    assert st["guarded_batches"] >= 1
    assert bits_equal(v, ref)


@pytest.mark.parametrize("kind", ["unaligned_rows", "coarse_voxels"])
def test_raw_device_entry_falls_back_to_packing(cuda, oracle, kind):
    """cbb_backproject_raw_device when the staged kernel cannot run -- rows
    not 16-byte aligned (W % 4 != 0) or footprint boxes over the budget
    (coarse voxels): it packs internally and runs the gather kernel, same
    bits as the reference."""
    import torch

    if kind == "unaligned_rows":
        cfg = synth.shrunk(synth.CONFIGS[2], edge_voxels=48, num_projections=12, width=1247,
                           height=960)
        g = VolumeGeometry.centered(48, 0.5)
    else:
        cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=48, num_projections=12)
        g = cfg.geometry
    _, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=12)
    n, H, W = imgs.shape
    assert pkg.tma_plan(g, W, H, 0, 48, mats)["staged"] == 0
    ref = np.zeros((48,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs.cpu().numpy(), mats) == 0
    flags = torch.zeros(n, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    pkg.scan_device(imgs, flags, err)
    v = torch.zeros((48, 48, 48), dtype=torch.float32, device="cuda")
    pkg.backproject_raw_device(v, g, 0, 48, imgs, W, H, n, mats, flags, pkg.Options(), err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0 and bits_equal(v.cpu().numpy(), ref)


def test_scan_flags_and_nonfinite(cuda):
    """scan_projections: bit 0 of a projection's flag when a pixel reaches
    2^86 (the exact division's numerator bound), err bit 2 on a non-finite
    pixel; unaligned sizes take the scalar loop."""
    import torch

    for w in (64, 63):
        x = torch.ones((4, 17, w), dtype=torch.float32, device="cuda")
        x[1, 3, 5] = 2.0 ** 86
        x[2, 16, w - 1] = -(2.0 ** 90)
        flags = torch.full((4,), 7, dtype=torch.int32, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        pkg.scan_device(x, flags, err)
        torch.cuda.synchronize()
        assert flags.tolist() == [0, 1, 1, 0] and int(err.item()) == 0
        x[3, 0, 0] = float("inf")
        pkg.scan_device(x, flags, err)
        torch.cuda.synchronize()
        assert int(err.item()) & 2


@pytest.mark.parametrize("resident", [True, False])
def test_pipeline_raw_mode_several_workers(scan, expected, monkeypatch, resident):
    """Raw mode with 3 slab workers on the one GPU: each keeps its band of
    raw rows (the uploading worker copies its band out of its slot, the others
    copy theirs from it), scans and back-projects them -- bitwise; with a
    forced guarded batch too."""
    g, mats, imgs = scan
    if not resident:
        monkeypatch.setenv("CBB_NO_RESIDENT", "1")
    host = imgs.cpu().numpy()
    v = np.zeros((L, L, L), np.float32)
    st = pkg.reconstruct_arrays(v, g, host, mats, pkg.Options(device_ids=[0, 0, 0], batch=8))
    assert st["num_gpus"] == 3
    assert bits_equal(v, expected)
    monkeypatch.setenv("CBB_FORCE_GUARDED", "1")
    v = np.zeros((L, L, L), np.float32)
    st = pkg.reconstruct_arrays(v, g, host, mats, pkg.Options(device_ids=[0, 0], batch=16))
    assert st["guarded_batches"] > 0 and bits_equal(v, expected)

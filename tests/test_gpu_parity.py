"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors. Exact mode must be BITWISE equal; fast mode must
meet north_star's tolerance (relL2 <= 1e-5, max|d| <= 1e-4 * range)."""
import numpy as np
import pytest

from conftest import bits_equal, load_golden

import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200 import synth
from paper_1401_3615_b200.geometry import VolumeGeometry

pytestmark = pytest.mark.gpu

REL_L2_TOL = 1e-5      # north_star
MAX_ABS_TOL = 1e-4     # x (max r - min r), north_star


def rel_l2(v, r):
    v = v.astype(np.float64)
    r = r.astype(np.float64)
    return float(np.linalg.norm(v - r) / max(np.linalg.norm(r), 1e-300))


def max_abs_over_range(v, r):
    rng = float(r.max() - r.min()) or 1.0
    return float(np.abs(v.astype(np.float64) - r).max() / rng)


def gpu_reconstruct(geom, mats, imgs, vol0, **opt):
    vol = pkg.Volume(geom, vol0.copy())
    st = pkg.reconstruct(vol, pkg.ProjectionStack(geom, mats, imgs), pkg.Options(**opt))
    return vol.voxels, st


def test_golden_hash_on_gpu(cuda, oracle):
    # proj/tests/test_kernel_ref.cpp:236-269 through the B200 kernel
    g, mats, imgs = oracle.golden_case()
    v, st = gpu_reconstruct(g, mats, imgs, np.zeros((64, 64, 64), np.float32))
    assert oracle.fnv1a64(v) == oracle.GOLDEN_HASH
    assert st["voxel_updates"] == 64 ** 3 * 32


@pytest.mark.parametrize("name", ["mini_c0.npz", "random_w.npz", "orthographic.npz"])
def test_reference_fixtures_bitwise(cuda, name):
    g, mats, imgs, vol0, expected = load_golden(name)
    v, st = gpu_reconstruct(g, mats, imgs, vol0)
    assert bits_equal(v, expected)
    if name == "random_w.npz":
        assert st["guarded_batches"] > 0  # w changes sign: guarded kernel ran


@pytest.mark.parametrize("batch", [1, 5, 32])
def test_batch_size_does_not_change_a_bit(cuda, batch):
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    v, _ = gpu_reconstruct(g, mats, imgs, vol0, batch=batch)
    assert bits_equal(v, expected)


def test_culling_is_exact(cuda):
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    on, _ = gpu_reconstruct(g, mats, imgs, vol0, cull=True)
    off, _ = gpu_reconstruct(g, mats, imgs, vol0, cull=False)
    assert bits_equal(on, expected) and bits_equal(off, expected)


def test_negative_zero_voxels_keep_reference_semantics(cuda, oracle):
    # -0.0 + (+0) = +0 in the reference; culling must not skip that update
    g, mats, imgs, vol0, _ = load_golden("mini_c0.npz")
    v0 = vol0.copy()
    v0[::2, ::3, :] = -0.0
    ref = v0.copy()
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    for mode_cull in (True, False):
        v, _ = gpu_reconstruct(g, mats, imgs, v0, cull=mode_cull)
        assert bits_equal(v, ref)


def test_cpp_adapter_with_reference_types(cuda):
    """oracle/_ref/adapter_golden: the reference's own types and generators
    (golden case) through include/conebeam_b200.hpp -> libconebeam_b200.so,
    compared with the reference's reconstruct_reference (built here from
    /root/reference; the binary travels with the snapshot)."""
    import subprocess

    import oracle as O

    exe = O.os.path.join(O.HERE, "_ref", "adapter_golden")
    if not O.os.path.exists(exe):
        pytest.skip("adapter_golden not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "reference ab67551f9fba3780 b200 ab67551f9fba3780" in out.stdout
    assert "validation nan 1 short 1 padded 1" in out.stdout


@pytest.mark.parametrize("where", [0, 7777, -1])
def test_c_abi_rejects_non_finite_voxels(cuda, where):
    """Volume::validate (proj/src/dataset.cpp:146-151, run by
    backproject_reference, kernel_ref.cpp:7) at the C ABI itself: every
    host-pointer entry point given a volume with one NaN / Inf voxel returns
    CBB_ERR_INVALID (status 1, the reference's validation_error) with the
    reference's message, and leaves the caller's volume untouched. The
    Python wrappers' own host-side validation is bypassed."""
    import ctypes as C

    from paper_1401_3615_b200 import _lib
    from paper_1401_3615_b200.backproject import geometry_c

    g, mats, imgs, vol0, _ = load_golden("mini_c0.npz")
    L = g.edge_voxels
    bad = vol0.copy()
    bad.reshape(-1)[where] = np.nan if where != 7777 else np.inf
    lib = _lib.lib()
    gc = geometry_c(g)
    imgs = np.ascontiguousarray(imgs)
    m = np.ascontiguousarray(mats, np.float64)
    N, H, W = imgs.shape

    def expect_invalid(status, v):
        assert status == 1, status
        assert lib.cbb_last_error().decode() == "Volume contains non-finite values"
        assert bits_equal(v, bad)

    for ids in ([0], [0, 0]):
        oc, _keep = pkg.Options(device_ids=ids, batch=8).to_c()
        v = bad.copy()
        expect_invalid(lib.cbb_reconstruct(v.ctypes.data, C.byref(gc), imgs.ctypes.data, W, H, N,
                                           m.ctypes.data, C.byref(oc), None), v)
        ptrs = (C.c_void_p * N)(*[imgs[i].ctypes.data for i in range(N)])
        v = bad.copy()
        expect_invalid(lib.cbb_reconstruct_images(v.ctypes.data, C.byref(gc), ptrs, W, H, N,
                                                  m.ctypes.data, C.byref(oc), None), v)
        h = C.c_void_p()
        expect_invalid(lib.cbb_session_create(C.byref(gc), W, H, bad.ctypes.data, C.byref(oc),
                                              C.byref(h)), bad)
        assert not h.value
    v = bad.copy()
    expect_invalid(lib.cbb_backproject(v.ctypes.data, C.byref(gc), imgs[0].ctypes.data, W, H,
                                       m.ctypes.data), v)
    # volume_is_zero: the caller promised zeros, nothing is read or checked
    oc, _keep = pkg.Options(num_gpus=1, volume_is_zero=True).to_c()
    v = bad.copy()
    assert lib.cbb_reconstruct(v.ctypes.data, C.byref(gc), imgs.ctypes.data, W, H, N,
                               m.ctypes.data, C.byref(oc), None) == 0
    # a bad image is reported first, as reconstruct_reference validates the
    # stack before the volume (kernel_ref.cpp:33)
    badimg = imgs.copy()
    badimg[3, 5, 5] = np.nan
    oc, _keep = pkg.Options(num_gpus=1).to_c()
    v = bad.copy()
    assert lib.cbb_reconstruct(v.ctypes.data, C.byref(gc), badimg.ctypes.data, W, H, N,
                               m.ctypes.data, C.byref(oc), None) == 1
    assert lib.cbb_last_error().decode() == "ProjectionImage contains non-finite values"
    assert L > 0


def test_per_projection_entry_point(cuda):
    # backproject_reference semantics, one call per projection
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    vol = pkg.Volume(g, vol0.copy())
    for i in range(len(mats)):
        pkg.backproject(vol, imgs[i], mats[i])
    assert bits_equal(vol.voxels, expected)


def test_session_streaming(cuda):
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    with pkg.Session(g, imgs.shape[2], imgs.shape[1], vol0, pkg.Options(batch=4)) as s:
        for i in range(3):
            s.backproject(imgs[i], mats[i])
        part, _ = s.finish()  # flushes; the session keeps accumulating
        for i in range(3, len(mats)):
            s.backproject(imgs[i], mats[i])
        out, st = s.finish()
    assert bits_equal(out, expected)
    ref_part = vol0.copy()
    import oracle as O
    O.reconstruct(ref_part, g, imgs[:3], mats[:3])
    assert bits_equal(part, ref_part)


def test_device_api_slabs(cuda):
    import torch

    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    L = g.edge_voxels
    n, H, W = imgs.shape
    _, _, nb = pkg.packed_layout(W, H)
    raw = torch.from_numpy(imgs).cuda()
    packed = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
    pkg.pack_device(raw, packed)
    vol = torch.from_numpy(vol0.copy()).cuda()
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    bounds = [0, 5, 6, 17, L]  # uneven slabs, incl. a 1-plane slab
    for z0, z1 in zip(bounds[:-1], bounds[1:]):
        pkg.backproject_device(vol[z0:z1], g, z0, z1, packed, W, H, n, mats, err_flag=err)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert bits_equal(vol.cpu().numpy(), expected)


def test_distributed_driver_single_rank(cuda):
    """The torch.distributed z-slab driver (NCCL path at N > 1) with the CUDA
    hooks, at world size 1: double-buffered uploads from pinned memory, pack,
    back-projection, slab download -- bitwise vs the reference fixture."""
    import torch

    from paper_1401_3615_b200.distributed import DistributedReconstructor

    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    n, H, W = imgs.shape
    rec = DistributedReconstructor(g, W, H, batch=4)
    host = torch.from_numpy(imgs).pin_memory()
    slab = rec.reconstruct(host, mats, initial_slab=vol0)
    assert bits_equal(slab, expected)
    assert bits_equal(rec.gather(slab), expected)


@pytest.mark.parametrize("z0,z1", [(0, 9), (24, 40), (56, 64)])
def test_distributed_driver_row_band_slab(cuda, oracle, z0, z1):
    """The torch.distributed driver owning one narrow slab packs only its row
    band (cbb_row_band_for_slab -> cbb_pack_device_band ->
    cbb_backproject_device_band): bitwise the oracle's planes; a NaN in a row
    outside the band is still caught by the uploading rank's full scan."""
    import torch

    from paper_1401_3615_b200.distributed import DistributedReconstructor

    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=64, num_projections=30)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=15)
    imgs = imgs_t.numpy()
    ref = np.zeros((64,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    band = pkg.row_band_for_slab(g, cfg.width, cfg.height, z0, z1, mats)
    assert band.raw_rows < cfg.height
    rec = DistributedReconstructor(g, cfg.width, cfg.height, batch=8, slabs=[(z0, z1)])
    slab = rec.reconstruct(torch.from_numpy(imgs).pin_memory(), mats)
    assert bits_equal(slab, ref[z0:z1])
    bad = imgs.copy()
    row = 0 if band.raw_row0 > 0 else cfg.height - 1
    bad[9, row, 3] = np.inf
    with pytest.raises(pkg.ValidationError):
        rec.reconstruct(torch.from_numpy(bad).pin_memory(), mats)


def test_single_process_multi_worker_slabs(cuda):
    """cbb_reconstruct with several workers (one z-slab each): device_ids
    [0, 0, 0] runs three independent slab pipelines on one GPU (no kernel
    waits on another), exercising the multi-GPU host logic -- bitwise."""
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    for ids in ([0, 0], [0, 0, 0]):
        v, st = gpu_reconstruct(g, mats, imgs, vol0, device_ids=ids, batch=4)
        assert st["num_gpus"] == len(ids)
        assert bits_equal(v, expected)


def test_config4_geometry_bitwise(cuda, oracle):
    """BASELINE config 4 scan (360 deg, R 1000 / SDD 1500 mm, 1536x1536 at
    0.2 mm, 30 ellipsoids) on a 64^3 volume and 90 of its projections."""
    cfg = synth.shrunk(synth.CONFIGS[4], edge_voxels=64, num_projections=90)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=15)
    imgs = imgs_t.numpy()
    ref = np.zeros((64,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref))
    assert st["guarded_batches"] == 0
    assert bits_equal(v, ref)


def test_reconstruct_file_streaming(cuda, tmp_path):
    """CBPS file -> cbb_reconstruct_file (streamed from disk, batch 4) is
    bitwise the reference fixture; a NaN pixel is rejected like
    ProjectionStack::validate (proj/src/dataset.cpp:123-144)."""
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    p = str(tmp_path / "mini.cbps")
    pkg.write_stack(p, pkg.ProjectionStack(g, mats, imgs))
    vol, st = pkg.reconstruct_file(p, pkg.Options(batch=4), initial=pkg.Volume(g, vol0.copy()))
    assert bits_equal(vol.voxels, expected)
    assert st["voxel_updates"] == g.edge_voxels ** 3 * len(mats)
    bad = imgs.copy()
    bad[3, 5, 7] = np.nan
    raw = bytearray(open(p, "rb").read())
    off = 40 + 3 * (96 + 4 * imgs.shape[1] * imgs.shape[2]) + 96 + 4 * (5 * imgs.shape[2] + 7)
    raw[off:off + 4] = np.float32(np.nan).tobytes()
    open(p, "wb").write(bytes(raw))
    keep = vol0.copy()
    v2 = pkg.Volume(g, vol0.copy())
    with pytest.raises(pkg.ValidationError):
        pkg.reconstruct_file(p, initial=v2)
    assert bits_equal(v2.voxels, keep)


@pytest.mark.parametrize("ids", [[0], [0, 0]])
def test_resident_tail_overlap_bitwise(cuda, oracle, monkeypatch, ids):
    """cbb_reconstruct keeps every packed projection resident and computes a
    dense tail of each slab after the stream (overlapping the head's D2H):
    bitwise the same as the streaming-only pipeline (CBB_NO_RESIDENT) and the
    oracle, with one and two slab workers, ragged batches."""
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=64, num_projections=70)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=35)
    imgs = imgs_t.numpy()
    ref = np.zeros((64,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    monkeypatch.setenv("CBB_NO_RESIDENT", "1")
    plain, _ = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), device_ids=ids, batch=16)
    monkeypatch.delenv("CBB_NO_RESIDENT")
    for frac in ("0.05", "0.12", "0.5"):
        monkeypatch.setenv("CBB_TAIL_FRAC", frac)
        v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), device_ids=ids, batch=16)
        assert st["guarded_batches"] == 0
        assert bits_equal(v, plain)
        assert bits_equal(v, ref)


def _bands_from_trace(err: str):
    """(rows held, cells packed, cells total) per worker from CBB_TRACE lines."""
    import re
    out = []
    for m in re.finditer(r"rows \[(-?\d+), (-?\d+)\) cells (\d+) of (\d+)", err):
        out.append((int(m.group(2)) - int(m.group(1)), int(m.group(3)), int(m.group(4))))
    return out


@pytest.mark.parametrize("ids,filt,peer", [([0, 0, 0, 0], False, True), ([0, 0, 0], True, True),
                                           ([0, 0, 0, 0, 0], True, True),
                                           ([0, 0, 0, 0], False, False),
                                           ([0, 0, 0], True, False)])
def test_row_bands_and_rotating_roots_bitwise(cuda, oracle, monkeypatch, capfd, ids, filt, peer):
    """Several slab workers: batch k is uploaded once by worker k mod G and the
    others pack only the detector rows their slab projects onto, reading the
    root's slot over peer memory (peer) or after a strided band copy (here all
    workers share one device). Bitwise equal to the oracle, with and without
    the in-pipeline ramp filter (then vs one worker)."""
    if not peer:
        monkeypatch.setenv("CBB_NO_PEER_PACK", "1")
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=64, num_projections=45)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=15)
    imgs = imgs_t.numpy()
    monkeypatch.setenv("CBB_TRACE", "1")
    if filt:
        opt = dict(ramp_filter_pixel_mm=cfg.pixel_mm)
        ref, _ = gpu_reconstruct(g, mats, imgs, np.zeros((64,) * 3, np.float32),
                                 device_ids=[0], **opt)
        capfd.readouterr()
    else:
        opt = {}
        ref = np.zeros((64,) * 3, np.float32)
        assert oracle.reconstruct(ref, g, imgs, mats) == 0
    v, st = gpu_reconstruct(g, mats, imgs, np.zeros((64,) * 3, np.float32), device_ids=ids,
                            batch=8, **opt)
    bands = _bands_from_trace(capfd.readouterr().err)
    assert len(bands) == len(ids)
    assert all(cells < total for _, cells, total in bands)  # every slab packs a band
    assert st["num_gpus"] == len(ids)
    assert bits_equal(v, ref)
    # pageable source: staged through the pinned double buffer, same bits
    v2, _ = gpu_reconstruct(g, mats, np.array(imgs, copy=True), np.zeros_like(v),
                            device_ids=ids, batch=5, **opt)
    assert bits_equal(v2, ref)


@pytest.mark.parametrize("ids", [[0], [0, 0]])
def test_nan_in_rows_no_band_holds_is_rejected(cuda, ids):
    """A 32 mm volume projects onto ~160 of the 960 detector rows, so every
    worker's row band skips row 5; the uploading root still scans the whole
    batch and a NaN there is rejected like ProjectionStack::validate
    (proj/src/dataset.cpp:123-144), leaving the volume untouched."""
    cfg = synth.shrunk(synth.CONFIGS[0], num_projections=12)
    g0, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=12)
    g = VolumeGeometry.centered(32, 1.0)
    imgs = imgs_t.numpy().copy()
    imgs[7, 5, 100] = np.nan
    vol = pkg.Volume(g, np.full((32,) * 3, 2.0, np.float32))
    with pytest.raises(pkg.ValidationError):
        pkg.reconstruct(vol, pkg.ProjectionStack(g, mats, imgs),
                        pkg.Options(device_ids=ids, batch=4))
    assert np.all(vol.voxels == 2.0)


def test_culled_update_counters(cuda):
    """cbb_run_stats.culled_updates: (voxel, projection) pairs skipped by warp
    culling. Never more than the pairs whose position is off the detector
    (ix <= -2, ix >= W, iy <= -2 or iy >= H, counted here in float64), most
    of them (> 25 % here) when the volume overhangs the field of view, and 0 with culling
    off; the volume is bitwise the same either way."""
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=64, num_projections=24)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=12)
    imgs = imgs_t.numpy()
    L = g.edge_voxels
    zero = np.zeros((L,) * 3, np.float32)
    v_on, st_on = gpu_reconstruct(g, mats, imgs, zero, cull=True, device_ids=[0, 0],
                                  count_culled=True)
    v_off, st_off = gpu_reconstruct(g, mats, imgs, zero, cull=False, count_culled=True)
    v_nc, st_nc = gpu_reconstruct(g, mats, imgs, zero)
    assert bits_equal(v_on, v_off) and bits_equal(v_on, v_nc)
    assert st_off["culled_updates"] == 0 and st_off["culled_fraction"] == 0.0
    assert st_nc["culled_fraction"] == -1.0
    idx = g.origin_mm + np.arange(L) * g.voxel_mm
    Z, Y, X = np.meshgrid(idx, idx, idx, indexing="ij")
    hom = np.stack([X.ravel(), Y.ravel(), Z.ravel(), np.ones(X.size)])
    off = 0
    for a in mats:
        u, v, w = a.reshape(4, 3).T @ hom
        ix, iy = u / w, v / w
        off += int(np.count_nonzero((ix <= -2) | (ix >= cfg.width) | (iy <= -2) | (iy >= cfg.height)))
    assert 0 < st_on["culled_updates"] <= off
    assert st_on["culled_updates"] > 0.25 * off, (st_on["culled_updates"], off)
    assert st_on["culled_fraction"] == pytest.approx(st_on["culled_updates"] / st_on["voxel_updates"])


@pytest.mark.parametrize("ids", [[0], [0, 0, 0]])
def test_reconstruct_images_separate_buffers(cuda, ids):
    """cbb_reconstruct_images (one buffer per projection, as the reference's
    ProjectionStack holds them): bitwise the reference fixture; a null image
    pointer or a NaN pixel is rejected and leaves the volume untouched."""
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    parts = [np.array(imgs[i], copy=True) for i in range(len(imgs))]
    v = vol0.copy()
    st = pkg.reconstruct_images(v, g, parts, mats, pkg.Options(device_ids=ids, batch=4))
    assert bits_equal(v, expected)
    assert st["voxel_updates"] == g.edge_voxels ** 3 * len(mats)
    parts[len(parts) // 2][1, 2] = np.nan
    v2 = vol0.copy()
    with pytest.raises(pkg.ValidationError):
        pkg.reconstruct_images(v2, g, parts, mats, pkg.Options(device_ids=ids))
    assert bits_equal(v2, vol0)


@pytest.mark.parametrize("resident", [True, False])
def test_w_zero_inside_slab_leaves_volume(cuda, monkeypatch, resident):
    """w == 0 exactly on plane z = 20 of a 32^3 volume (w = world z): the
    guarded kernel flags it and cbb_reconstruct raises GeometryError before
    writing any plane, whether or not the resident tail pass is used."""
    if not resident:
        monkeypatch.setenv("CBB_NO_RESIDENT", "1")
    g = VolumeGeometry(32, 1.0, -20.0)
    m = np.zeros((3, 12))
    m[:, 0] = m[:, 4] = 1.0
    m[:, 8] = 1.0
    m[:, 9] = m[:, 10] = 4.0
    imgs = np.ones((3, 16, 16), np.float32)
    vol = pkg.Volume(g, np.full((32, 32, 32), 3.0, np.float32))
    with pytest.raises(pkg.GeometryError):
        pkg.reconstruct(vol, pkg.ProjectionStack(g, m, imgs))
    assert np.all(vol.voxels == 3.0)


def test_fast_mode_within_tolerance(cuda):
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    v, _ = gpu_reconstruct(g, mats, imgs, vol0, mode=pkg.MODE_FAST)
    assert rel_l2(v, expected) <= REL_L2_TOL
    assert max_abs_over_range(v, expected) <= MAX_ABS_TOL


def test_w_zero_raises_and_leaves_volume(cuda):
    # proj/tests/test_kernel_ref.cpp:224-234
    g = VolumeGeometry.centered(4, 1.0)
    m = np.zeros(12)
    m[0] = m[4] = 1.0
    vol = pkg.Volume(g, np.full((4, 4, 4), 3.0, np.float32))
    with pytest.raises(pkg.GeometryError):
        pkg.backproject(vol, np.ones((8, 8), np.float32), m)
    assert np.all(vol.voxels == 3.0)


def test_zero_image_and_validation(cuda):
    g = VolumeGeometry.centered(8, 1.0)
    vol = pkg.Volume(g, np.arange(512, dtype=np.float32).reshape(8, 8, 8))
    before = vol.voxels.copy()
    m = np.zeros(12)
    m[0] = m[4] = 1.0
    m[9] = m[10] = 8.0
    m[11] = 1.0
    pkg.backproject(vol, np.zeros((16, 16), np.float32), m)
    assert bits_equal(vol.voxels, before)
    bad = np.zeros((16, 16), np.float32)
    bad[3, 3] = np.nan
    with pytest.raises(pkg.ValidationError):
        pkg.backproject(vol, bad, m)
    with pytest.raises(pkg.GeometryError):
        pkg.reconstruct(pkg.Volume(VolumeGeometry.centered(9, 1.0)),
                        pkg.ProjectionStack(g, m[None], np.zeros((1, 16, 16), np.float32)))


@pytest.mark.parametrize("L,W,H", [(1, 1, 1), (37, 19, 11), (33, 1, 40), (9, 64, 1)])
def test_ragged_sizes(cuda, oracle, L, W, H):
    r = synth.SplitMix64(L * 1000 + W * 10 + H)
    g = VolumeGeometry.centered(L, 2.0)
    cfg = pkg.TrajectoryConfig(7, 200.0, 400.0, W, H, 160.0 / max(W, H))
    mats = pkg.make_circular_trajectory(cfg)
    imgs = np.array([r.uniform(-3, 3) for _ in range(7 * W * H)], np.float32).reshape(7, H, W)
    vol0 = np.array([r.uniform(-1, 1) for _ in range(L ** 3)], np.float32).reshape(L, L, L)
    ref = vol0.copy()
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    v, _ = gpu_reconstruct(g, mats, imgs, vol0, batch=3)
    assert bits_equal(v, ref)


def test_seeded_random_matrices_guarded_path(cuda, oracle):
    # reference-test-style random stacks (proj/tests/helpers.hpp:59-93)
    r = synth.SplitMix64(7)
    done = 0
    for trial in range(40):
        L = 1 + int(r.uniform(0, 12))
        g = VolumeGeometry(L, r.uniform(0.1, 2.0), r.uniform(-10.0, 10.0))
        n = 1 + int(r.uniform(0, 4))
        W = 1 + int(r.uniform(0, 16))
        H = 1 + int(r.uniform(0, 16))
        mats = np.array([[r.uniform(-5, 5) for _ in range(12)] for _ in range(n)])
        imgs = np.array([r.uniform(-100, 100) for _ in range(n * H * W)],
                        np.float32).reshape(n, H, W)
        vol0 = np.array([r.uniform(-100, 100) for _ in range(L ** 3)],
                        np.float32).reshape(L, L, L)
        ref = vol0.copy()
        s = oracle.reconstruct(ref, g, imgs, mats)
        if s != 0:
            continue
        v, _ = gpu_reconstruct(g, mats, imgs, vol0)
        assert bits_equal(v, ref), f"trial {trial}"
        done += 1
    assert done >= 20


def test_config0_geometry_bitwise(cuda, oracle):
    """BASELINE config 0 scan (128^3 @ 2 mm, 1248x960 @ 0.32 mm, 200 deg) on
    62 of its projections, bitwise against the oracle."""
    cfg = synth.shrunk(synth.CONFIGS[0], num_projections=62)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=31)
    imgs = imgs_t.numpy()
    ref = np.zeros((128,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref))
    assert st["guarded_batches"] == 0
    assert bits_equal(v, ref)
    fv, _ = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), mode=pkg.MODE_FAST)
    assert rel_l2(fv, ref) <= REL_L2_TOL and max_abs_over_range(fv, ref) <= MAX_ABS_TOL


def test_large_detector_integer_cell_indices(cuda, oracle, monkeypatch):
    """A 3600 x 2800 detector (packed grid 3696 x 2896 = 10.7M cells, past the
    2^23 of the float cell index): the integer-index kernels -- fast path,
    counting instantiation, guarded kernel -- bitwise against the oracle."""
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=48, num_projections=8, width=3600,
                       height=2800)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=4)
    imgs = imgs_t.numpy()
    assert pkg.packed_layout(3600, 2800)[0] * pkg.packed_layout(3600, 2800)[1] > 2 ** 23
    ref = np.zeros((48,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    assert np.count_nonzero(ref) > 0.5 * ref.size
    v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref))
    assert st["guarded_batches"] == 0
    assert bits_equal(v, ref)
    v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), count_culled=1)
    assert bits_equal(v, ref)
    fv, _ = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), mode=pkg.MODE_FAST)
    assert rel_l2(fv, ref) <= REL_L2_TOL and max_abs_over_range(fv, ref) <= MAX_ABS_TOL
    monkeypatch.setenv("CBB_FORCE_GUARDED", "1")
    v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref))
    assert st["guarded_batches"] > 0
    assert bits_equal(v, ref)


@pytest.mark.slow
def test_config2_full_size_planes_bitwise(cuda, oracle):
    """Full BASELINE config 2 (512^3, 496 x 1248x960): whole volume on the
    GPU through the device path; the oracle recomputes a few z-planes
    (top, centre, bottom) and they must match bitwise. Also checks the
    size-independent additivity property over a split stack."""
    import torch

    cfg = synth.CONFIGS[2]
    g, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=16)
    L, (n, H, W) = g.edge_voxels, imgs.shape
    _, _, nb = pkg.packed_layout(W, H)
    packed = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
    pkg.pack_device(imgs, packed)
    vol = torch.zeros((L, L, L), dtype=torch.float32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    pkg.backproject_device(vol, g, 0, L, packed, W, H, n, mats, err_flag=err)
    # additivity: same stack in two calls (248 + 248) is bitwise identical
    vol2 = torch.zeros_like(vol)
    pkg.backproject_device(vol2, g, 0, L, packed, W, H, 248, mats[:248], err_flag=err)
    pkg.backproject_device(vol2, g, 0, L, packed, W, H, 248, mats[248:], err_flag=err,
                           first=248)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert bool(torch.equal(vol.view(torch.int32), vol2.view(torch.int32)))
    host = imgs.cpu().numpy()
    for z0 in (0, 255, 511):
        slab = np.zeros((1, L, L), np.float32)
        assert oracle.reconstruct_slab(slab, g, z0, z0 + 1, host, mats) == 0
        assert bits_equal(vol[z0:z0 + 1].cpu().numpy(), slab), f"plane {z0}"


def test_texture_side_variant_is_close_not_exact(cuda, oracle):
    """cbb_backproject_texture_device (north_star's hardware-texture side
    number): 8-bit texture weights and floor addressing put it near, not at,
    the reference -- relL2 0.05-0.15 (coarser grids err more), far above
    the 1e-5 parity bar, so it is only ever reported beside the exact
    result."""
    import torch

    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=48, num_projections=40)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=20)
    imgs = imgs_t.numpy()
    ref = np.zeros((48,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    vt = torch.zeros((48,) * 3, dtype=torch.float32, device="cuda")
    raw = torch.from_numpy(imgs).cuda()
    for _ in range(2):  # second call reuses the cached layered array
        vt.zero_()
        pkg.backproject_texture_device(vt, g, 0, 48, raw, mats)
    torch.cuda.synchronize()
    v = vt.cpu().numpy()
    e = rel_l2(v, ref)
    assert 1e-5 < e < 0.3, e
    # cached arrays / buffers are freed on request and rebuilt on demand
    pkg.release_cached_memory()
    v2, _ = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref))
    assert bits_equal(v2, ref)


@pytest.mark.slow
def test_config0_and_config1_full_volumes_bitwise(cuda, oracle):
    """BASELINE configs 0 (128^3) and 1 (256^3), all 496 projections, through
    the host C ABI (pinned input, two slab workers for config 1): the whole
    volume bitwise against the threaded oracle."""
    for cid, ids in ((0, [0]), (1, [0, 0])):
        cfg = synth.CONFIGS[cid]
        g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=62)
        imgs = imgs_t.numpy()
        L = g.edge_voxels
        ref = np.zeros((L,) * 3, np.float32)
        assert oracle.reconstruct(ref, g, imgs, mats) == 0
        v = np.zeros_like(ref)
        st = pkg.reconstruct_arrays(v, g, imgs, mats, pkg.Options(device_ids=ids))
        assert st["voxel_updates"] == L ** 3 * 496 and st["guarded_batches"] == 0
        assert bits_equal(v, ref), f"config {cid}"


@pytest.mark.slow
@pytest.mark.parametrize("cid,count", [(3, 496), (4, 180)])
def test_1024_volumes_planes_bitwise(cuda, oracle, cid, count):
    """The 1024^3 volumes (4 GiB): config 3 (496 x 1248x960) and config 4's
    detector and trajectory (1536x1536, 360 deg; first 180 of its 1440
    projections) through cbb_reconstruct into a pinned host volume with the
    resident tail; the oracle recomputes the bottom, centre and top planes."""
    import torch

    cfg = synth.CONFIGS[cid]
    g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=30,
                                      count=count, pin=True)
    L = g.edge_voxels
    vol_t = torch.zeros((L, L, L), dtype=torch.float32).pin_memory()
    v = vol_t.numpy()
    st = pkg.reconstruct_arrays(v, g, imgs.numpy(), mats, pkg.Options(volume_is_zero=True))
    assert st["voxel_updates"] == L ** 3 * count
    host = imgs.numpy()
    for z0 in (0, L // 2, L - 1):
        slab = np.zeros((1, L, L), np.float32)
        assert oracle.reconstruct_slab(slab, g, z0, z0 + 1, host, mats) == 0
        assert bits_equal(v[z0:z0 + 1], slab), f"config {cid} plane {z0}"


@pytest.mark.parametrize("scale_exp", [105, 90, -75, 0])
def test_extreme_pixel_magnitudes_take_the_exact_fallback(cuda, oracle, scale_exp):
    """The fast correctly-rounded weight division is proven for nonzero
    |val| in [2^-60, 2^86). Projections scaled by 2^105 or 2^90 (flagged per
    projection by pack_quads' metadata word) or 2^-75 (caught by the kernel's
    minimum tracking) must take the IEEE-division fallback and stay bitwise
    equal to the reference; mixed with ordinary projections."""
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=32, num_projections=24)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=12)
    imgs = imgs_t.numpy().astype(np.float64)
    imgs[5] *= 2.0 ** scale_exp
    imgs[17] *= 2.0 ** scale_exp
    imgs = imgs.astype(np.float32)
    assert np.all(np.isfinite(imgs))
    ref = np.zeros((32,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    for ids in ([0], [0, 0]):
        v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), device_ids=ids, batch=8)
        assert bits_equal(v, ref), (scale_exp, ids)


@pytest.mark.parametrize("mscale", [1000.0, 2.0 ** -15, 2.0 ** 19])
def test_scaled_matrices_stay_on_the_fast_kernels(cuda, oracle, mscale):
    """Calibrated matrices are often not normalised to w ~ 1 (mm-scaled P has
    w ~ 500-1500). The fast kernels' divisions are proven for w in
    [2^-20, 2^20] (runtime_common.cuh: projection_is_safe), so such stacks
    run unguarded and stay bitwise equal to the reference, mixed with an
    ordinary pixel range and with pixels near the 2^86 numerator bound."""
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=40, num_projections=20)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=10)
    imgs = imgs_t.numpy().copy()
    mats = mats * mscale
    for big in (False, True):
        if big:
            imgs[3] = (imgs[3].astype(np.float64) * 2.0 ** 80).astype(np.float32)
        ref = np.zeros((40,) * 3, np.float32)
        assert oracle.reconstruct(ref, g, imgs, mats) == 0
        for ids in ([0], [0, 0]):
            v, st = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), device_ids=ids, batch=8)
            assert st["guarded_batches"] == 0, (mscale, ids)
            assert bits_equal(v, ref), (mscale, big, ids)


@pytest.mark.parametrize("name", ["mini_c0.npz", "orthographic.npz"])
def test_guarded_kernel_equals_fast_path(cuda, monkeypatch, name):
    """proj/tests/test_kernel_ref.cpp:51-65 restated for the two kernels: the
    guarded kernel (scalar IEEE divisions, reference guards; used when the
    host cannot prove a batch safe) and the unguarded fast path give the
    same bits, both equal to the reference fixture."""
    g, mats, imgs, vol0, expected = load_golden(name)
    v_fast, st_fast = gpu_reconstruct(g, mats, imgs, vol0)
    monkeypatch.setenv("CBB_FORCE_GUARDED", "1")
    v_guard, st_guard = gpu_reconstruct(g, mats, imgs, vol0)
    assert st_fast["guarded_batches"] == 0 and st_guard["guarded_batches"] > 0
    assert bits_equal(v_fast, expected) and bits_equal(v_guard, expected)


def test_affine_field_reproduced_and_within_tap_hull(cuda, oracle):
    """proj/tests/test_kernel_ref.cpp:67-115 restated on the GPU path: with an
    affine projection field (the golden 'ramp' ix + 2 iy), voxels that project
    inside the detector in every view get exactly the field's values, so the
    volume matches a float64 evaluation of sum_p (ix + 2 iy) / w^2 to 1e-4
    relative there; and a single projection's update lies within the hull of
    its four taps scaled by 1/w^2."""
    g, mats, imgs = oracle.golden_case()
    v, _ = gpu_reconstruct(g, mats, imgs, np.zeros((64,) * 3, np.float32))
    L = g.edge_voxels
    idx = g.origin_mm + np.arange(L) * g.voxel_mm
    Z, Y, X = np.meshgrid(idx, idx, idx, indexing="ij")
    hom = np.stack([X.ravel(), Y.ravel(), Z.ravel(), np.ones(X.size)])
    acc = np.zeros(X.size)
    inside = np.ones(X.size, bool)
    for a in mats:
        u, vv, w = a.reshape(4, 3).T @ hom
        ix, iy = u / w, vv / w
        inside &= (ix > 0.01) & (iy > 0.01) & (ix < 158.99) & (iy < 158.99)
        acc += (ix + 2.0 * iy) / (w * w)
    assert inside.sum() > 0.2 * X.size
    got = v.ravel().astype(np.float64)[inside]
    err = np.abs(got - acc[inside]).max() / np.abs(acc[inside]).max()
    assert err < 1e-4, err
    # one projection: the update at every interior voxel lies within its taps' hull
    one, _ = gpu_reconstruct(g, mats[:1], imgs[:1], np.zeros((64,) * 3, np.float32))
    u, vv, w = mats[0].reshape(4, 3).T @ hom
    fx, fy = u / w, vv / w
    ok = (fx > 0.01) & (fy > 0.01) & (fx < 158.99) & (fy < 158.99)
    ix, iy = np.floor(fx), np.floor(fy)
    lo = (ix + 2.0 * iy) / (w * w)
    hi = (ix + 1 + 2.0 * (iy + 1)) / (w * w)
    o = one.ravel().astype(np.float64)
    assert np.all(o[ok] >= lo[ok] * (1 - 1e-5) - 1e-6)
    assert np.all(o[ok] <= hi[ok] * (1 + 1e-5) + 1e-6)


def test_single_process_slabs_are_work_balanced(cuda, oracle, monkeypatch, capfd):
    """cbb_reconstruct with 4 workers and the whole stack known: the z-slabs
    are split by estimated (non-culled) work, so the outer slabs, whose planes
    leave the field of view, hold more planes; the result stays bitwise."""
    import re

    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=64, num_projections=30)
    g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=15)
    imgs = imgs_t.numpy()
    ref = np.zeros((64,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, imgs, mats) == 0
    monkeypatch.setenv("CBB_TRACE", "1")
    capfd.readouterr()
    v, _ = gpu_reconstruct(g, mats, imgs, np.zeros_like(ref), device_ids=[0, 0, 0, 0])
    err = capfd.readouterr().err
    slabs = sorted({(int(a), int(b)) for a, b in re.findall(r"slab \[(\d+), (\d+)\) rows", err)})
    assert len(slabs) == 4 and slabs[0][0] == 0 and slabs[-1][1] == 64
    assert all(slabs[i][1] == slabs[i + 1][0] for i in range(3))
    sizes = [b - a for a, b in slabs]
    assert sizes[0] > sizes[1] and sizes[3] > sizes[2], sizes
    assert bits_equal(v, ref)


def test_resume_from_partial_volume_is_bitwise(cuda):
    """Checkpoint / resume: reconstruct the first part of a
    stack, save the volume (CBPV round trip), continue with the rest on top
    of it -- bitwise the single-call result, as in the reference's additivity
    test (proj/tests/test_kernel_ref.cpp:190-222)."""
    import tempfile

    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    k = len(mats) // 3
    part = pkg.Volume(g, vol0.copy())
    pkg.reconstruct(part, pkg.ProjectionStack(g, mats[:k], imgs[:k]))
    with tempfile.TemporaryDirectory() as d:
        path = d + "/part.cbpv"
        pkg.write_volume(path, part)
        resumed = pkg.read_volume(path)
    pkg.reconstruct(resumed, pkg.ProjectionStack(g, mats[k:], imgs[k:]))
    assert bits_equal(resumed.voxels, expected)


def test_plain_c_example_runs_on_the_gpu(cuda, tmp_path):
    """examples/reconstruct_c.c end to end: plain C, cbb_reconstruct on the GPU."""
    import os
    import shutil
    import subprocess

    from conftest import ROOT

    if shutil.which("gcc") is None:
        pytest.skip("no gcc on this box")
    exe = str(tmp_path / "reconstruct_c")
    lib = os.path.join(ROOT, "paper_1401_3615_b200")
    subprocess.run(["gcc", "-std=c99", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "reconstruct_c.c"), "-L" + lib,
                    "-lconebeam_b200", "-Wl,-rpath," + lib, "-lm", "-o", exe],
                   check=True, capture_output=True, timeout=120)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "voxel updates" in out.stdout
    assert 'nan voxel: status 1 "Volume contains non-finite values" (volume unchanged)' in out.stdout


def test_concurrent_calls_from_host_threads(cuda, oracle):
    """cbb_reconstruct from four host threads at once (ctypes releases the
    GIL): each call owns its streams, the buffer caches are locked, so every
    result is bitwise the sequential one."""
    import threading

    cases = []
    for k in range(4):
        cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=40 + 8 * k, num_projections=20 + 3 * k)
        g, mats, imgs_t = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=10)
        imgs = imgs_t.numpy()
        ref = np.zeros((g.edge_voxels,) * 3, np.float32)
        assert oracle.reconstruct(ref, g, imgs, mats) == 0
        cases.append((g, mats, imgs, ref))
    out = [None] * len(cases)
    errors = []

    def run(i):
        try:
            g, mats, imgs, _ = cases[i]
            for _ in range(3):
                v = np.zeros((g.edge_voxels,) * 3, np.float32)
                pkg.reconstruct_arrays(v, g, np.array(imgs), mats,
                                       pkg.Options(device_ids=[0] * (1 + i % 2), batch=7))
            out[i] = v
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    for (g, mats, imgs, ref), v in zip(cases, out):
        assert bits_equal(v, ref)

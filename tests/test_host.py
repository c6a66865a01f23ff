"""CPU: host-side logic -- geometry conventions, file formats, generator
determinism, the C-ABI library's exported surface (no compute calls)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200 import synth
from paper_1401_3615_b200.geometry import (TrajectoryConfig, VolumeGeometry, dehomogenize,
                                           forward_project, make_circular_trajectory)


def small_config(n=1, rng=2.0 * math.pi):
    return TrajectoryConfig(n, 750.0, 1200.0, 1248, 960, 0.32, rng)


# --- geometry (restates proj/tests/test_geometry.cpp:172-271) -----------------

def test_trajectory_isocenter_normalised_and_centred():
    for m in make_circular_trajectory(small_config(17)):
        u, v, w = forward_project(m, 0.0, 0.0, 0.0)
        assert abs(w - 1.0) <= 1e-9
        ix, iy = dehomogenize(u, v, w)
        assert abs(ix - 623.5) <= 1e-6 and abs(iy - 479.5) <= 1e-6


def test_trajectory_matches_pinhole_oracle():
    c = small_config(5, 3.0)
    ms = make_circular_trajectory(c)
    r = synth.SplitMix64(4242)
    for i, m in enumerate(ms):
        ang = c.angular_range_rad * i / c.num_projections
        cs, sn = math.cos(ang), math.sin(ang)
        R, f = c.source_isocenter_mm, c.source_detector_mm / c.pixel_size_mm
        cu, cv = 0.5 * (c.detector_width - 1), 0.5 * (c.detector_height - 1)
        rot = np.array([[-sn, cs, 0.0], [0.0, 0.0, 1.0], [-cs, -sn, 0.0]])
        src = np.array([R * cs, R * sn, 0.0])
        K = np.array([[f, 0, cu], [0, f, cv], [0, 0, 1.0]])
        P = np.hstack([K @ rot, (-K @ rot @ src)[:, None]])
        P /= P[2, 3]
        for _ in range(50):
            x, y, z = (r.uniform(-80, 80) for _ in range(3))
            got = forward_project(m, x, y, z)
            want = P @ np.array([x, y, z, 1.0])
            assert np.allclose(got, want, rtol=1e-9, atol=1e-9)


def test_geometry_validation():
    with pytest.raises(pkg.ValidationError):
        VolumeGeometry(0, 1.0, 0.0).validate()
    with pytest.raises(pkg.ValidationError):
        VolumeGeometry(8, -1.0, 0.0).validate()
    c = small_config()
    c.detector_width = 0
    with pytest.raises(pkg.ValidationError, match="detector_width"):
        make_circular_trajectory(c)
    with pytest.raises(pkg.GeometryError):
        dehomogenize(1.0, 1.0, 0.0)


def test_centered_origin():
    g = VolumeGeometry.centered(512, 0.5)
    assert g.origin_mm == -127.75


# --- file formats (restates proj/tests/test_dataset.cpp:33-128) ---------------

def two_image_stack():
    mats = np.zeros((2, 12))
    mats[:, 11] = 1.0
    mats[0, 0], mats[1, 0] = 1.0, 2.0
    imgs = np.stack([np.full((3, 4), float(i), np.float32) for i in range(2)])
    return pkg.ProjectionStack(VolumeGeometry(4, 1.0, -1.5), mats, imgs)


def test_stack_file_size_and_roundtrip(tmp_path):
    p = str(tmp_path / "s.cbps")
    pkg.write_stack(p, two_image_stack())
    header = 4 + 2 + 2 + 4 + 4 + 4 + 8 + 8 + 4
    assert os.path.getsize(p) == header + 2 * (12 * 8 + 4 * 3 * 4)
    s = pkg.read_stack(p)
    p2 = str(tmp_path / "s2.cbps")
    pkg.write_stack(p2, s)
    assert open(p, "rb").read() == open(p2, "rb").read()


def test_volume_file_roundtrip(tmp_path):
    v = pkg.Volume(VolumeGeometry(3, 0.7, -2.0),
                   np.arange(27, dtype=np.float32).reshape(3, 3, 3) * 0.5)
    p = str(tmp_path / "v.cbpv")
    pkg.write_volume(p, v)
    assert os.path.getsize(p) == 4 + 2 + 2 + 4 + 8 + 8 + 27 * 4
    w = pkg.read_volume(p)
    assert np.array_equal(w.voxels, v.voxels) and w.geometry == v.geometry


def test_file_corruption_cases(tmp_path):
    p = str(tmp_path / "s.cbps")
    pkg.write_stack(p, two_image_stack())
    raw = bytearray(open(p, "rb").read())
    bad = bytearray(raw)
    bad[0:4] = b"SPBC"
    open(p, "wb").write(bad)
    with pytest.raises(pkg.FormatError):
        pkg.read_stack(p)
    bad = bytearray(raw)
    bad[4] = 9
    open(p, "wb").write(bad)
    with pytest.raises(pkg.FormatError):
        pkg.read_stack(p)
    open(p, "wb").write(raw[:-7])
    with pytest.raises(pkg.TruncatedError):
        pkg.read_stack(p)
    open(p, "wb").write(raw + b"\0")
    with pytest.raises(pkg.FormatError):
        pkg.read_stack(p)
    with pytest.raises(pkg.IOError_):
        pkg.read_stack(str(tmp_path / "missing.cbps"))


# --- generator ---------------------------------------------------------------

def test_splitmix64_known_values():
    # splitmix64 reference outputs for seed 1234567
    r = synth.SplitMix64(1234567)
    assert [r.next_u64() for _ in range(3)] == [6457827717110365317, 3203168211198807973,
                                                9817491932198370423]


def test_generator_is_deterministic_and_border_heavy():
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=16, num_projections=3, width=156,
                       height=120)
    g1, m1, i1 = synth.make_inputs(cfg)
    g2, m2, i2 = synth.make_inputs(cfg)
    assert np.array_equal(m1, m2) and bool((i1 == i2).all())
    # perturbed matrices keep the w(0) == 1 normalisation
    for m in m1:
        assert abs(forward_project(m, 0, 0, 0)[2] - 1.0) < 1e-12
    im = i1.numpy()
    assert np.abs(im[:, :, 0]).mean() > 1.2 * np.abs(im[:, :, 78]).mean()


def test_baseline_config_arithmetic():
    assert synth.CONFIGS[0].voxel_updates == 128 ** 3 * 496
    assert synth.CONFIGS[2].voxel_updates == 512 ** 3 * 496
    assert synth.CONFIGS[4].voxel_updates == 1024 ** 3 * 1440


# --- the C ABI ----------------------------------------------------------------

def header_functions():
    text = open(os.path.join(ROOT, "include", "conebeam_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cbb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_1401_3615_b200 import _lib

    L = _lib.lib()
    names = header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTS)


def test_status_names_and_layout_without_gpu():
    from paper_1401_3615_b200 import _lib

    L = _lib.lib()
    assert L.cbb_status_name(0) == b"ok"
    assert L.cbb_status_name(5) == b"geometry error"
    qp, qr, nb = pkg.packed_layout(1248, 960)
    # kPad = 48 cells of zero margin on each side (rows padded to 8 cells)
    # plus one 16-byte metadata cell per projection
    assert qp % 8 == 0 and qp >= 1248 + 96 and qr == 960 + 96 and nb == qp * qr * 16 + 16
    with pytest.raises(pkg.ValidationError):
        pkg.packed_layout(0, 10)
    # past 2^23 cells the kernels form integer cell indices; the layout stays
    qp, qr, nb = pkg.packed_layout(3600, 2800)
    assert qp * qr > 2 ** 23 and nb == qp * qr * 16 + 16
    with pytest.raises(pkg.ValidationError):  # kMagic + cell index must fit int32
        pkg.packed_layout(40000, 40000)


def test_struct_layouts_match_header():
    from paper_1401_3615_b200 import _lib

    assert ctypes.sizeof(_lib.VolumeGeometryC) == 24
    assert ctypes.sizeof(_lib.OptionsC) == 64
    assert ctypes.sizeof(_lib.RunStatsC) == 8 * 4 + 8 * 2 + 8 + 8 * 8 + 8 + 8
    assert ctypes.sizeof(_lib.StackFileInfoC) == 40


# --- CBPS header through the C ABI (host-only code path) -------------------------

def test_stack_file_query_matches_reader(tmp_path):
    s = two_image_stack()
    p = str(tmp_path / "q.cbps")
    pkg.write_stack(p, s)
    info = pkg.stack_file_info(p)
    assert info == {"edge_voxels": 4, "voxel_mm": 1.0, "origin_mm": -1.5, "count": 2,
                    "width": 4, "height": 3}


def test_stack_file_query_error_mapping(tmp_path):
    # same exception classes as read_stack (proj/tests/test_dataset.cpp:76-128)
    p = str(tmp_path / "e.cbps")
    pkg.write_stack(p, two_image_stack())
    raw = bytearray(open(p, "rb").read())
    cases = [(b"SPBC" + raw[4:], pkg.FormatError), (raw[:4] + b"\x09" + raw[5:], pkg.FormatError),
             (raw[:-7], pkg.TruncatedError), (raw + b"\0", pkg.FormatError),
             (raw[:20], pkg.TruncatedError)]
    for data, exc in cases:
        open(p, "wb").write(bytes(data))
        with pytest.raises(exc):
            pkg.stack_file_info(p)
    with pytest.raises(pkg.IOError_):
        pkg.stack_file_info(str(tmp_path / "missing.cbps"))


def test_row_bands_cover_every_tap():
    """cbb_row_band_for_slab (host-side, no GPU): for 8 z-slabs of a scan, the
    band's cell rows contain the cell of every voxel x projection tap the
    kernel can read (trunc(iy), clamped to [-2, H] off the margin), its raw
    rows every detector row those cells hold, and it is narrower than the
    detector; a projection with w <= 0 on the slab gives the full detector."""
    import paper_1401_3615_b200 as pkg
    from paper_1401_3615_b200 import synth

    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=64, num_projections=62)
    g = cfg.geometry
    mats = synth.perturbed_matrices(cfg)
    W, H = cfg.width, cfg.height
    qp, qr, _ = pkg.packed_layout(W, H)
    pad = (qr - H) // 2
    L = g.edge_voxels
    rng = np.random.default_rng(3)
    for z0 in range(0, L, 8):
        z1 = z0 + 8
        b = pkg.row_band_for_slab(g, W, H, z0, z1, mats)
        assert b.cell_rows < qr
        idx = rng.integers(0, L, size=(3000, 2))
        zi = rng.integers(z0, z1, size=3000)
        corners = np.array([[x, y, z] for x in (0, L - 1) for y in (0, L - 1) for z in (z0, z1 - 1)])
        pts = np.concatenate([np.stack([idx[:, 0], idx[:, 1], zi], 1), corners])
        wpt = g.origin_mm + pts * g.voxel_mm
        hom = np.concatenate([wpt, np.ones((len(pts), 1))], 1)
        for a in mats:
            A = a.reshape(4, 3).T  # column-major 3x4
            u, v, w = A @ hom.T
            assert np.all(w > 0)
            iy = np.trunc(v / w)
            inside = (iy >= -pad) & (iy <= H + pad - 2)
            cell = np.where(inside, iy, np.clip(iy, -2, H)) + pad
            assert cell.min() >= b.cell_row0 and cell.max() < b.cell_row0 + b.cell_rows
        rows_needed = [r for c in range(b.cell_row0 - pad, b.cell_row0 + b.cell_rows - pad)
                       for r in (c, c + 1) if 0 <= r < H]
        if rows_needed:
            assert min(rows_needed) >= b.raw_row0
            assert max(rows_needed) < b.raw_row0 + b.raw_rows
    bad = mats.copy()
    bad[5, 11] = -5.0  # w(0) < 0 for projection 5
    full = pkg.row_band_for_slab(g, W, H, 0, 8, bad)
    assert (full.raw_row0, full.raw_rows, full.cell_row0, full.cell_rows) == (0, H, 0, qr)


def test_c_abi_from_plain_c(tmp_path):
    """include/conebeam_b200.h is plain C99: examples/reconstruct_c.c compiles
    with -Wall -Wextra -Werror against it, links libconebeam_b200.so and runs
    (ABI part only: no GPU here)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    exe = str(tmp_path / "reconstruct_c")
    lib = os.path.join(ROOT, "paper_1401_3615_b200")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror",
           "-I" + os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "reconstruct_c.c"),
           "-L" + lib, "-lconebeam_b200", "-Wl,-rpath," + lib, "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, timeout=120)
    out = subprocess.run([exe, "--abi-only"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "geometry error" in out.stdout


def test_abi_rejects_invalid_inputs_before_touching_the_gpu():
    """Argument validation of the C ABI runs before any CUDA call, so it is
    checked here without a GPU: empty stacks, zero sizes, non-finite
    matrices, bad options, oversize detectors and null pointers give
    CBB_ERR_INVALID (1) with the reference's messages; the volume is not
    touched."""
    import ctypes as C

    from paper_1401_3615_b200 import _lib
    from paper_1401_3615_b200.backproject import geometry_c

    L = _lib.lib()
    g = geometry_c(pkg.VolumeGeometry.centered(8, 1.0))
    vol = np.full((8, 8, 8), 7.0, np.float32)
    imgs = np.zeros((2, 4, 5), np.float32)
    mats = np.zeros((2, 12))
    mats[:, 0] = mats[:, 4] = mats[:, 11] = 1.0

    def call(geom=g, w=5, h=4, n=2, m=mats, opt=None, v=vol, im=imgs):
        oc = _lib.OptionsC()
        L.cbb_options_defaults(C.byref(oc))
        for k, val in (opt or {}).items():
            setattr(oc, k, val)
        st = L.cbb_reconstruct(None if v is None else v.ctypes.data, C.byref(geom),
                               None if im is None else im.ctypes.data, w, h, n,
                               m.ctypes.data, C.byref(oc), None)
        return st, L.cbb_last_error().decode()

    assert call(n=0) == (1, "ProjectionStack: at least one projection required")
    assert call(w=0)[0] == 1 and "dimensions" in call(w=0)[1]
    assert call(h=-3)[0] == 1
    assert call(w=40000, h=40000)[0] == 1 and "too large" in call(w=40000, h=40000)[1]
    bad = mats.copy()
    bad[1, 7] = np.nan
    assert call(m=bad) == (1, "ProjectionMatrix: field 'a[7]' must be finite")
    assert call(geom=geometry_c(pkg.VolumeGeometry(0, 1.0, 0.0)))[0] == 1
    assert call(opt={"batch": 0})[0] == 1 and "batch" in call(opt={"batch": 0})[1]
    assert call(opt={"batch": 65})[0] == 1
    assert call(opt={"mode": 7})[0] == 1
    assert call(opt={"slab_begin": 5, "slab_end": 3})[0] == 1
    assert call(opt={"ramp_filter": 1, "filter_pixel_mm": 0.0})[0] == 1
    assert call(v=None)[0] == 1 and "null" in call(v=None)[1]
    assert call(im=None)[0] == 1
    ids = (C.c_int32 * 1)(0)
    assert call(opt={"device_ids": C.cast(ids, C.POINTER(C.c_int32)), "num_gpus": 0}) == (
        1, "options: device_ids needs num_gpus > 0 (its length)")
    assert np.all(vol == 7.0)


def test_array_entry_points_check_sizes_before_the_library():
    """reconstruct_arrays / reconstruct_images hand raw pointers to the C ABI,
    which reads one matrix per image and L^3 voxels: mismatched sizes raise
    ValidationError first."""
    g = pkg.VolumeGeometry.centered(8, 1.0)
    imgs = np.zeros((3, 4, 5), np.float32)
    mats = np.zeros((3, 12))
    mats[:, 0] = mats[:, 4] = mats[:, 11] = 1.0
    with pytest.raises(pkg.ValidationError, match="L\\^3"):
        pkg.reconstruct_arrays(np.zeros(100, np.float32), g, imgs, mats)
    with pytest.raises(pkg.ValidationError, match="differ in length"):
        pkg.reconstruct_arrays(np.zeros((8, 8, 8), np.float32), g, imgs, mats[:2])
    with pytest.raises(pkg.ValidationError, match="L\\^3"):
        pkg.reconstruct_images(np.zeros(7, np.float32), g, list(imgs), mats)
    with pytest.raises(pkg.ValidationError, match="differ in length"):
        pkg.reconstruct_images(np.zeros((8, 8, 8), np.float32), g, list(imgs), mats[:1])


def test_tma_plan_for_baseline_configs(monkeypatch):
    """Host-side staging plan of the TMA kernel (cbb_tma_plan, no GPU): the
    0.5 / 0.25 mm configs (2, 3, 4) stage their footprint boxes in shared
    memory; the coarse 2 mm / 1 mm volumes (configs 0, 1: boxes over the
    budget), detectors whose rows are not 16-byte aligned and
    CBB_BP_PATH=quad take the packed-quad kernel."""
    for cid, staged in ((0, 0), (1, 0), (2, 1), (3, 1), (4, 1)):
        cfg = synth.CONFIGS[cid]
        m = synth.perturbed_matrices(cfg)
        g = cfg.geometry
        p = pkg.tma_plan(g, cfg.width, cfg.height, 0, g.edge_voxels, m)
        assert p["staged"] == staged, (cid, p)
        if staged:
            assert p["box_width"] >= p["footprint_width"] and p["box_width"] % 16 == 0
            assert p["box_rows"] >= p["footprint_rows"] and 3 <= p["stages"] <= 8
    cfg = synth.CONFIGS[2]
    m = synth.perturbed_matrices(cfg)
    assert pkg.tma_plan(cfg.geometry, 1247, 960, 0, 512, m)["staged"] == 0
    monkeypatch.setenv("CBB_BP_PATH", "quad")
    assert pkg.tma_plan(cfg.geometry, 1248, 960, 0, 512, m)["staged"] == 0


def test_options_default_to_one_gpu():
    """cbb_options_defaults: one GPU unless asked (the cross-device paths are
    tested with several workers on one GPU only), exact mode, batch 32."""
    import ctypes as C

    from paper_1401_3615_b200 import _lib

    oc = _lib.OptionsC()
    _lib.lib().cbb_options_defaults(C.byref(oc))
    assert (oc.num_gpus, oc.batch, oc.mode, oc.cull) == (1, 32, 0, 1)
    o, _keep = pkg.Options(device_ids=[0, 0]).to_c()
    assert o.num_gpus == 2

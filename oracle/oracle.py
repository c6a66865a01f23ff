"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU checkers.

  * liboracle.so             -- fdk_oracle.c, the C restatement of the
                                reference oracle (proj/include/conebeam/kernel_ref.hpp:19-70,
                                proj/src/kernel_ref.cpp:5-38).
  * _ref/libconebeam_ref.so  -- the reference's own sources compiled by
                                oracle/Makefile (+ ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module, and only as the checker or the timed reference
CPU implementation; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libconebeam_ref.so")

GOLDEN_HASH = 0xAB67551F9FBA3780  # proj/tests/test_kernel_ref.cpp:264

_oracle = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.oracle_bilinear_sample_guarded.restype = C.c_float
        L.oracle_bilinear_sample_guarded.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_float,
                                                     C.c_float]
        L.oracle_backproject.restype = C.c_int
        L.oracle_backproject.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                         C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.oracle_reconstruct.restype = C.c_int
        L.oracle_reconstruct.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                         C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                         C.c_int]
        L.oracle_reconstruct_slab.restype = C.c_int
        L.oracle_reconstruct_slab.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                              C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                              C.c_int, C.c_void_p, C.c_int]
        L.oracle_reconstruct_planes.restype = C.c_int
        L.oracle_reconstruct_planes.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                                C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                                C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.oracle_content_hash.restype = C.c_uint64
        L.oracle_content_hash.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
        L.oracle_fnv1a64.restype = C.c_uint64
        L.oracle_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} absent (built from /root/reference by oracle/Makefile)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_reconstruct_reference.restype = C.c_int
        L.ref_reconstruct_reference.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                                C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                C.c_void_p]
        L.ref_backproject_reference.restype = C.c_int
        L.ref_backproject_reference.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double,
                                                C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.ref_reconstruct_optimized.restype = C.c_int
        L.ref_reconstruct_optimized.argtypes = [
            C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int, C.c_int, C.c_int,
            C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
            C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.ref_make_circular_trajectory.restype = C.c_int
        L.ref_make_circular_trajectory.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int,
                                                   C.c_int, C.c_double, C.c_double, C.c_void_p]
        L.ref_bilinear_sample_guarded.restype = C.c_float
        L.ref_bilinear_sample_guarded.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_float,
                                                  C.c_float]
        _ref = L
    return _ref


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def sample(img, ix: float, iy: float) -> float:
    im = _f32(img)
    return float(oracle_lib().oracle_bilinear_sample_guarded(im.ctypes.data, im.shape[1],
                                                             im.shape[0], ix, iy))


def reconstruct(vol: np.ndarray, geometry, imgs, mats, threads: int = 0) -> int:
    """oracle_reconstruct in place on vol (L,L,L) float32; returns the status
    (0 ok, 5 = w == 0 geometry error)."""
    assert vol.dtype == np.float32 and vol.flags.c_contiguous
    im = _f32(imgs)
    if im.ndim == 2:
        im = im[None]
    m = _f64(mats).reshape(-1, 12)
    threads = threads or (os.cpu_count() or 1)
    return int(oracle_lib().oracle_reconstruct(
        vol.ctypes.data, geometry.edge_voxels, geometry.voxel_mm, geometry.origin_mm,
        im.ctypes.data, im.shape[2], im.shape[1], im.shape[0], m.ctypes.data, threads))


def reconstruct_slab(vol_slab: np.ndarray, geometry, z_begin: int, z_end: int, imgs, mats,
                     threads: int = 0) -> int:
    """oracle_reconstruct_slab: planes [z_begin, z_end) of the L^3 volume."""
    assert vol_slab.dtype == np.float32 and vol_slab.flags.c_contiguous
    L = geometry.edge_voxels
    assert vol_slab.size == (z_end - z_begin) * L * L
    im = _f32(imgs)
    if im.ndim == 2:
        im = im[None]
    m = _f64(mats).reshape(-1, 12)
    threads = threads or (os.cpu_count() or 1)
    return int(oracle_lib().oracle_reconstruct_slab(
        vol_slab.ctypes.data, L, geometry.voxel_mm, geometry.origin_mm, int(z_begin),
        int(z_end), im.ctypes.data, im.shape[2], im.shape[1], im.shape[0], m.ctypes.data,
        threads))


def reconstruct_planes(out: np.ndarray, geometry, planes, imgs, mats, threads: int = 0) -> int:
    """oracle_reconstruct_planes: out (len(planes), L, L) float32 accumulates
    the listed z-planes of reconstruct_reference (cache-tiled, all threads)."""
    assert out.dtype == np.float32 and out.flags.c_contiguous
    L = geometry.edge_voxels
    pl = np.ascontiguousarray(planes, dtype=np.int32)
    assert out.size == pl.size * L * L
    im = _f32(imgs)
    if im.ndim == 2:
        im = im[None]
    m = _f64(mats).reshape(-1, 12)
    threads = threads or (os.cpu_count() or 1)
    return int(oracle_lib().oracle_reconstruct_planes(
        out.ctypes.data, L, geometry.voxel_mm, geometry.origin_mm, pl.ctypes.data, pl.size,
        im.ctypes.data, im.shape[2], im.shape[1], im.shape[0], m.ctypes.data, threads))


def content_hash(a: np.ndarray) -> int:
    b = np.ascontiguousarray(a)
    return int(oracle_lib().oracle_content_hash(b.ctypes.data, b.nbytes, os.cpu_count() or 1))


def cache_dir():
    """Directory of cached oracle planes (CBB_ORACLE_CACHE; "off" disables).
    A cache only saves time: a missing or damaged entry is recomputed, and
    nothing on a fresh GPU box depends on it."""
    d = os.environ.get("CBB_ORACLE_CACHE", os.path.join(os.path.expanduser("~"), ".cache",
                                                        "cbb_oracle"))
    return None if d == "off" else d


def reference_planes(geometry, planes, imgs, mats, threads: int = 0):
    """reconstruct_reference's z-planes `planes` of a zero-initialised volume
    (oracle_reconstruct_planes), cached on disk under a content hash of the
    inputs -- the reference bench's hash-keyed reference-volume cache
    (proj/src/bench.cpp:194-214). Returns (planes array, seconds computing,
    cache hit)."""
    import time

    pl = np.ascontiguousarray(planes, dtype=np.int32)
    im = _f32(imgs)
    m = _f64(mats).reshape(-1, 12)
    L = geometry.edge_voxels
    key = None
    d = cache_dir()
    if d:
        hdr = np.array([L, geometry.voxel_mm, geometry.origin_mm, *im.shape], np.float64)
        h = 0
        for part in (im, m, hdr, pl):
            h = ((h * 1099511628211) ^ content_hash(part)) & 0xFFFFFFFFFFFFFFFF
        key = "%016x" % h
        path = os.path.join(d, f"ref-{key}.npy")
        if os.path.exists(path):
            try:
                out = np.load(path)
                if out.shape == (pl.size, L, L) and out.dtype == np.float32:
                    return out, 0.0, True
            except (OSError, ValueError):
                pass  # stale or damaged entry: rebuild
    out = np.zeros((pl.size, L, L), np.float32)
    t0 = time.perf_counter()
    st = reconstruct_planes(out, geometry, pl, im, m, threads)
    secs = time.perf_counter() - t0
    if st != 0:
        raise RuntimeError(f"oracle_reconstruct_planes failed with status {st}")
    if key:
        try:
            os.makedirs(d, exist_ok=True)
            tmp = os.path.join(d, f".ref-{key}.{os.getpid()}.npy")
            np.save(tmp, out)
            os.replace(tmp, os.path.join(d, f"ref-{key}.npy"))
        except OSError:
            pass
    return out, secs, False


def fnv1a64(a: np.ndarray) -> int:
    b = np.ascontiguousarray(a)
    return int(oracle_lib().oracle_fnv1a64(b.ctypes.data, b.nbytes))


def ref_reconstruct_reference(vol: np.ndarray, geometry, imgs, mats) -> int:
    im = _f32(imgs)
    if im.ndim == 2:
        im = im[None]
    m = _f64(mats).reshape(-1, 12)
    return int(ref_lib().ref_reconstruct_reference(
        vol.ctypes.data, geometry.edge_voxels, geometry.voxel_mm, geometry.origin_mm,
        im.ctypes.data, im.shape[2], im.shape[1], im.shape[0], m.ctypes.data))


def ref_reconstruct_optimized(vol: np.ndarray, geometry, imgs, mats, lanes=16, chunk=262,
                              workers=0, use_clip=True, use_pad=True) -> dict:
    im = _f32(imgs)
    if im.ndim == 2:
        im = im[None]
    m = _f64(mats).reshape(-1, 12)
    pre, ker, upd = C.c_double(), C.c_double(), C.c_uint64()
    s = ref_lib().ref_reconstruct_optimized(
        vol.ctypes.data, geometry.edge_voxels, geometry.voxel_mm, geometry.origin_mm,
        im.ctypes.data, im.shape[2], im.shape[1], im.shape[0], m.ctypes.data, lanes, chunk,
        workers, int(use_clip), int(use_pad), C.byref(pre), C.byref(ker), C.byref(upd))
    return {"status": int(s), "precompute_seconds": pre.value, "kernel_seconds": ker.value,
            "voxel_updates": int(upd.value)}


def ref_trajectory(cfg) -> np.ndarray:
    out = np.empty((cfg.num_projections, 12), dtype=np.float64)
    s = ref_lib().ref_make_circular_trajectory(
        cfg.num_projections, cfg.source_isocenter_mm, cfg.source_detector_mm,
        cfg.detector_width, cfg.detector_height, cfg.pixel_size_mm, cfg.angular_range_rad,
        out.ctypes.data)
    if s != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return out


def ref_sample(img, ix: float, iy: float) -> float:
    im = _f32(img)
    return float(ref_lib().ref_bilinear_sample_guarded(im.ctypes.data, im.shape[1], im.shape[0],
                                                       ix, iy))


# ---- fixtures shared by tests and smoke ------------------------------------------

def golden_case():
    """The reference's golden reconstruction (proj/tests/test_kernel_ref.cpp:236-269):
    32 projections, SID 200, SDD 400, 160x160 px at 1 mm, full circle, matrices
    rounded to 1e-6, 64^3 at 1 mm, 'ramp' field p0*ix + p1*iy + p2 with
    defaults (1, 2, 0) (proj/src/dataset.cpp:262-263) evaluated in double and
    rounded to float."""
    from paper_1401_3615_b200.geometry import (TrajectoryConfig, VolumeGeometry,
                                               make_circular_trajectory)

    cfg = TrajectoryConfig(32, 200.0, 400.0, 160, 160, 1.0)
    mats = make_circular_trajectory(cfg)
    x = mats * 1e6  # std::round: half away from zero
    mats = np.sign(x) * np.floor(np.abs(x) + 0.5) / 1e6
    iy, ix = np.meshgrid(np.arange(160, dtype=np.float64), np.arange(160, dtype=np.float64),
                         indexing="ij")
    img = (1.0 * ix + 2.0 * iy + 0.0).astype(np.float32)
    imgs = np.broadcast_to(img, (32, 160, 160)).copy()
    geom = VolumeGeometry.centered(64, 1.0)
    return geom, mats, imgs

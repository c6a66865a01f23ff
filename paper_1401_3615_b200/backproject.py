"""Host-side mirror of the reference's back-projection interface, running on
the B200 through the C ABI of libconebeam_b200.so.

Reference interface                                 -> here
  backproject_reference(Volume&, img, matrix)         -> backproject(vol, img, matrix)
    (proj/include/conebeam/kernel_ref.hpp:77, proj/src/kernel_ref.cpp:5-30)
  reconstruct_reference(Volume&, stack)               -> reconstruct(vol, stack)
    (proj/src/kernel_ref.cpp:32-38)
  reconstruct_optimized(vol, stack, OptOptions, stats)-> reconstruct(vol, stack, options, ...)
    (proj/src/kernel_opt.cpp:658-716)
Same argument meaning and error behaviour: geometry mismatch and w == 0 raise
GeometryError, bad inputs raise ValidationError, the volume accumulates (+=).
In exact mode the result is bitwise that of reconstruct_reference.

There is no CPU path: every call goes through the CUDA library and raises if
it cannot be loaded or no device is present.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .dataset import ProjectionStack, Volume, check_same_geometry
from .errors import ValidationError
from .geometry import VolumeGeometry, validate_matrices

MODE_EXACT = 0
MODE_FAST = 1


@dataclass
class Options:
    """cbb_options (include/conebeam_b200.h); B200 counterpart of OptOptions
    (proj/include/conebeam/kernel_opt.hpp:121-133)."""

    num_gpus: int = 1                 # 0 = all visible devices
    device_ids: Optional[Sequence[int]] = None
    batch: int = 32                   # projections per pipeline batch (1..64)
    mode: int = MODE_EXACT
    cull: bool = True
    volume_is_zero: bool = False
    slab: Optional[Sequence[int]] = None  # (z_begin, z_end) planes to update; None = all
    ramp_filter_pixel_mm: Optional[float] = None  # set: inputs are raw line integrals, FDK-filter on GPU
    count_culled: bool = False        # run stats report culled updates (slower kernels)

    def to_c(self):
        o = _lib.OptionsC()
        _lib.lib().cbb_options_defaults(C.byref(o))
        o.num_gpus = int(self.num_gpus)
        keep = None
        if self.device_ids is not None:
            keep = (C.c_int32 * len(self.device_ids))(*[int(d) for d in self.device_ids])
            o.device_ids = C.cast(keep, C.POINTER(C.c_int32))
            o.num_gpus = len(self.device_ids)  # the C ABI reads num_gpus ids
        o.batch = int(self.batch)
        o.mode = int(self.mode)
        o.cull = int(bool(self.cull))
        o.volume_is_zero = int(bool(self.volume_is_zero))
        if self.slab is not None:
            o.slab_begin, o.slab_end = int(self.slab[0]), int(self.slab[1])
        if self.ramp_filter_pixel_mm is not None:
            o.ramp_filter = 1
            o.filter_pixel_mm = float(self.ramp_filter_pixel_mm)
        o.count_culled = int(bool(self.count_culled))
        return o, keep


def geometry_c(g: VolumeGeometry) -> _lib.VolumeGeometryC:
    return _lib.VolumeGeometryC(int(g.edge_voxels), float(g.voxel_mm), float(g.origin_mm))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _image(img) -> np.ndarray:
    a = np.ascontiguousarray(img, dtype=np.float32)
    if a.ndim != 2:
        raise ValidationError("ProjectionImage: expected a 2-D (height, width) array")
    return a


def backproject(vol: Volume, img, matrix, validate: bool = True) -> None:
    """Accumulates one projection into the volume, in place.

    Semantics of backproject_reference (proj/src/kernel_ref.cpp:5-30): the
    image and volume are validated (finite values), the matrix is cast to
    float, and a voxel with w == 0 raises GeometryError (on error the volume
    is left unchanged here; the reference leaves it partially updated).
    """
    im = _image(img)
    m = validate_matrices(matrix)
    if m.shape[0] != 1:
        raise ValidationError("backproject: expected one 3x4 matrix")
    if validate:
        if not np.isfinite(im).all():
            raise ValidationError("ProjectionImage contains non-finite values")
        vol.validate()
    g = geometry_c(vol.geometry)
    L = _lib.lib()
    _lib.check(L.cbb_backproject(_ptr(vol.voxels), C.byref(g), _ptr(im), im.shape[1],
                                 im.shape[0], _ptr(m)))


def reconstruct(vol: Volume, stack: ProjectionStack, options: Optional[Options] = None,
                validate: bool = True) -> dict:
    """Back-projects every projection of the stack, in order, into vol (+=).

    reconstruct_reference / cb_reconstruct_optimized semantics; returns the
    per-phase run statistics (cb_run_stats counterpart). Multi-GPU via
    options.num_gpus: z-slabs, one per device.
    """
    if validate:
        stack.validate()
        vol.validate()
    check_same_geometry(vol, stack, "reconstruct")
    opt = options or Options()
    oc, _keep = opt.to_c()
    g = geometry_c(vol.geometry)
    st = _lib.RunStatsC()
    L = _lib.lib()
    _lib.check(L.cbb_reconstruct(_ptr(vol.voxels), C.byref(g), _ptr(stack.images),
                                 stack.width, stack.height, stack.count,
                                 _ptr(stack.matrices), C.byref(oc), C.byref(st)))
    return st.to_dict()


def _check_sizes(voxels: np.ndarray, geometry: VolumeGeometry, n_mats: int, n_imgs: int) -> None:
    # the library trusts the pointers it is given: L^3 voxels are uploaded and
    # written back, one matrix is read per image (Volume::validate and
    # ProjectionStack::validate, proj/src/dataset.cpp:131-151)
    if voxels.size != int(geometry.edge_voxels) ** 3:
        raise ValidationError("Volume: voxel buffer length != L^3")
    if n_mats != n_imgs:
        raise ValidationError("ProjectionStack: images and matrices differ in length")


def reconstruct_arrays(voxels: np.ndarray, geometry: VolumeGeometry, images: np.ndarray,
                       matrices: np.ndarray, options: Optional[Options] = None) -> dict:
    """Array-level reconstruct without validation scans (bench e2e leg):
    voxels (L,L,L) float32 accumulated in place; images (N,H,W) float32 (pinned
    or pageable host memory); matrices (N,12) float64."""
    if voxels.dtype != np.float32 or not voxels.flags.c_contiguous:
        raise ValidationError("voxels must be C-contiguous float32")
    if images.dtype != np.float32 or not images.flags.c_contiguous or images.ndim != 3:
        raise ValidationError("images must be C-contiguous float32 (N, H, W)")
    m = validate_matrices(matrices)
    _check_sizes(voxels, geometry, m.shape[0], images.shape[0])
    opt = options or Options()
    oc, _keep = opt.to_c()
    g = geometry_c(geometry)
    st = _lib.RunStatsC()
    _lib.check(_lib.lib().cbb_reconstruct(voxels.ctypes.data, C.byref(g), images.ctypes.data,
                                          images.shape[2], images.shape[1], images.shape[0],
                                          _ptr(m), C.byref(oc), C.byref(st)))
    return st.to_dict()


def reconstruct_images(voxels: np.ndarray, geometry: VolumeGeometry, images: Sequence,
                       matrices: np.ndarray, options: Optional[Options] = None) -> dict:
    """cbb_reconstruct_images: like reconstruct_arrays, but each projection is
    its own (H, W) float32 array (the reference's one-buffer-per-image stack);
    nothing is concatenated on the host."""
    if voxels.dtype != np.float32 or not voxels.flags.c_contiguous:
        raise ValidationError("voxels must be C-contiguous float32")
    imgs = list(images)
    if not imgs:
        raise ValidationError("ProjectionStack: at least one projection required")
    h, w = imgs[0].shape
    for a in imgs:
        if a.dtype != np.float32 or not a.flags.c_contiguous or a.shape != (h, w):
            raise ValidationError("images must be C-contiguous float32 (H, W) arrays of one shape")
    m = validate_matrices(matrices)
    _check_sizes(voxels, geometry, m.shape[0], len(imgs))
    ptrs = (C.c_void_p * len(imgs))(*[a.ctypes.data for a in imgs])
    oc, _keep = (options or Options()).to_c()
    st = _lib.RunStatsC()
    _lib.check(_lib.lib().cbb_reconstruct_images(voxels.ctypes.data, C.byref(geometry_c(geometry)),
                                                 ptrs, w, h, len(imgs), _ptr(m), C.byref(oc),
                                                 C.byref(st)))
    return st.to_dict()


def stack_file_info(path: str) -> dict:
    """Header of a CBPS stack file (cbb_stack_file_query); raises IOError_,
    FormatError, TruncatedError like read_stack (proj/src/dataset.cpp:181-212)."""
    info = _lib.StackFileInfoC()
    _lib.check(_lib.lib().cbb_stack_file_query(str(path).encode(), C.byref(info)))
    return {k: getattr(info, k) for k, _ in info._fields_}


def reconstruct_file(path: str, options: Optional[Options] = None,
                     initial: Optional[Volume] = None) -> tuple:
    """Reconstructs a CBPS stack file, streaming its projections from disk
    (cbb_reconstruct_file). Returns (Volume, run stats); `initial` (same
    geometry) is accumulated into, like reconstruct()."""
    info = stack_file_info(path)
    g = VolumeGeometry(info["edge_voxels"], info["voxel_mm"], info["origin_mm"])
    vol = Volume(g) if initial is None else initial
    if vol.geometry != g:
        from .errors import GeometryError
        raise GeometryError("reconstruct_file: volume and stack geometries differ")
    oc, _keep = (options or Options()).to_c()
    st = _lib.RunStatsC()
    _lib.check(_lib.lib().cbb_reconstruct_file(_ptr(vol.voxels), str(path).encode(),
                                               C.byref(oc), C.byref(st)))
    return vol, st.to_dict()


class Session:
    """Streaming per-projection back-projection (cbb_session_*), the
    RabbitCT-style module interface: feed projections one by one, read the
    volume with finish()."""

    def __init__(self, geometry: VolumeGeometry, width: int, height: int,
                 initial_volume: Optional[np.ndarray] = None,
                 options: Optional[Options] = None):
        geometry.validate()
        self.geometry = geometry
        self.width = int(width)
        self.height = int(height)
        self._init = None
        if initial_volume is not None:
            self._init = np.ascontiguousarray(initial_volume, dtype=np.float32)
            if self._init.size != geometry.voxel_count:
                raise ValidationError("Session: initial volume must hold L^3 voxels")
        oc, self._keep = (options or Options()).to_c()
        g = geometry_c(geometry)
        h = C.c_void_p()
        _lib.check(_lib.lib().cbb_session_create(
            C.byref(g), self.width, self.height,
            None if self._init is None else _ptr(self._init), C.byref(oc), C.byref(h)))
        self._h = h

    def backproject(self, img, matrix) -> None:
        im = _image(img)
        if im.shape != (self.height, self.width):
            raise ValidationError("Session: image dimensions differ from the session's")
        m = validate_matrices(matrix)
        _lib.check(_lib.lib().cbb_session_backproject(self._h, _ptr(im), _ptr(m)))

    def finish(self) -> tuple:
        L = self.geometry.edge_voxels
        out = np.empty((L, L, L), dtype=np.float32)
        st = _lib.RunStatsC()
        _lib.check(_lib.lib().cbb_session_finish(self._h, _ptr(out), C.byref(st)))
        return out, st.to_dict()

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().cbb_session_free(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --- device-resident path (torch tensors as plain device memory) ---------------

def release_cached_memory() -> None:
    """Frees the library's cached device/pinned buffers and texture arrays
    (cbb_release_cached_memory), like torch.cuda.empty_cache."""
    _lib.check(_lib.lib().cbb_release_cached_memory())


def packed_layout(width: int, height: int) -> tuple:
    """(quad_pitch, quad_rows, bytes_per_projection) of the packed gather layout."""
    qp, qr, nb = C.c_int32(), C.c_int32(), C.c_int64()
    _lib.check(_lib.lib().cbb_packed_layout(int(width), int(height), C.byref(qp), C.byref(qr),
                                            C.byref(nb)))
    return qp.value, qr.value, nb.value


def pack_device(raw, packed, stream=None) -> None:
    """raw: CUDA float32 tensor (N, H, W); packed: CUDA tensor with at least
    N * bytes_per_projection bytes. Enqueued on `stream` (torch stream or None
    for the current stream)."""
    import torch

    if not (raw.is_cuda and raw.dtype == torch.float32 and raw.is_contiguous() and raw.dim() == 3):
        raise ValidationError("pack_device: raw must be a contiguous CUDA float32 (N, H, W) tensor")
    n, h, w = raw.shape
    _, _, nb = packed_layout(w, h)
    if packed.numel() * packed.element_size() < n * nb:
        raise ValidationError("pack_device: packed buffer too small")
    s = stream if stream is not None else torch.cuda.current_stream(raw.device)
    _lib.check(_lib.lib().cbb_pack_device(raw.data_ptr(), w, h, n, packed.data_ptr(),
                                          C.c_void_p(s.cuda_stream)))


@dataclass(frozen=True)
class RowBand:
    """Detector rows [raw_row0, raw_row0 + raw_rows) a z-slab's voxels can
    touch, and the packed cell rows [cell_row0, cell_row0 + cell_rows) holding
    them (cbb_row_band_for_slab)."""
    raw_row0: int
    raw_rows: int
    cell_row0: int
    cell_rows: int

    def c(self):
        return _lib.RowBandC(self.raw_row0, self.raw_rows, self.cell_row0, self.cell_rows)

    def packed_bytes(self, width: int, height: int) -> int:
        qp, qr, nb = packed_layout(width, height)
        return qp * self.cell_rows * 16 + (nb - qp * qr * 16)  # cells + metadata cell


def row_band_for_slab(geometry: VolumeGeometry, width: int, height: int, z_begin: int,
                      z_end: int, matrices: np.ndarray) -> RowBand:
    """Row band of slab [z_begin, z_end) over these projections."""
    m = validate_matrices(matrices)
    b = _lib.RowBandC()
    _lib.check(_lib.lib().cbb_row_band_for_slab(C.byref(geometry_c(geometry)), int(width),
                                                int(height), int(z_begin), int(z_end), _ptr(m),
                                                m.shape[0], C.byref(b)))
    return RowBand(b.raw_row0, b.raw_rows, b.cell_row0, b.cell_rows)


def pack_device_band(raw, band: RowBand, packed, err_flag=None, stream=None,
                     height: Optional[int] = None) -> None:
    """Packs the band's cell rows of raw projections (cbb_pack_device_band).
    raw: CUDA float32 (N, rows, W) holding detector rows from band.raw_row0 on
    -- either the full detector (rows == height; pass height=None) or just the
    band (rows == band.raw_rows; pass the detector height)."""
    import torch

    if not (raw.is_cuda and raw.dtype == torch.float32 and raw.is_contiguous() and raw.dim() == 3):
        raise ValidationError("pack_device_band: raw must be a contiguous CUDA float32 (N, R, W) tensor")
    n, rows, w = raw.shape
    h = rows if height is None else int(height)
    ptr = raw.data_ptr()
    if height is None:  # full buffer: start at the band's first row
        ptr += band.raw_row0 * w * 4
    if packed.numel() * packed.element_size() < n * band.packed_bytes(w, h):
        raise ValidationError("pack_device_band: packed buffer too small")
    s = stream if stream is not None else torch.cuda.current_stream(raw.device)
    _lib.check(_lib.lib().cbb_pack_device_band(
        ptr, rows * w, w, h, n, C.byref(band.c()), packed.data_ptr(),
        None if err_flag is None else err_flag.data_ptr(), C.c_void_p(s.cuda_stream)))


def check_finite_device(values, err_flag, stream=None) -> None:
    """Sets bit 2 of err_flag (device int32) if a value is not finite."""
    import torch

    if not (values.is_cuda and values.dtype == torch.float32 and values.is_contiguous()):
        raise ValidationError("check_finite_device: contiguous CUDA float32 tensor")
    s = stream if stream is not None else torch.cuda.current_stream(values.device)
    _lib.check(_lib.lib().cbb_check_finite_device(values.data_ptr(), values.numel(),
                                                  err_flag.data_ptr(), C.c_void_p(s.cuda_stream)))


def backproject_device(vol_slab, geometry: VolumeGeometry, z_begin: int, z_end: int, packed,
                       width: int, height: int, count: int, matrices: np.ndarray,
                       options: Optional[Options] = None, err_flag=None, stream=None,
                       first: int = 0, band: Optional[RowBand] = None) -> None:
    """Enqueues the back-projection of `count` packed projections (starting at
    packed projection `first`) into a device z-slab [z_begin, z_end); with
    `band`, the projections were packed by pack_device_band with that band."""
    import torch

    if not (vol_slab.is_cuda and vol_slab.dtype == torch.float32 and vol_slab.is_contiguous()):
        raise ValidationError("backproject_device: vol_slab must be a contiguous CUDA float32 tensor")
    L = geometry.edge_voxels
    if vol_slab.numel() < (z_end - z_begin) * L * L:
        raise ValidationError("backproject_device: slab tensor too small")
    m = validate_matrices(matrices)
    if m.shape[0] < count:
        raise ValidationError("backproject_device: fewer matrices than projections")
    _, _, nb = packed_layout(width, height)
    oc, _keep = (options or Options()).to_c()
    g = geometry_c(geometry)
    s = stream if stream is not None else torch.cuda.current_stream(vol_slab.device)
    err = None if err_flag is None else err_flag.data_ptr()
    if band is None:
        _lib.check(_lib.lib().cbb_backproject_device(
            vol_slab.data_ptr(), C.byref(g), int(z_begin), int(z_end),
            packed.data_ptr() + int(first) * nb, int(width), int(height), int(count), _ptr(m),
            C.byref(oc), err, C.c_void_p(s.cuda_stream)))
        return
    nbb = band.packed_bytes(width, height)
    _lib.check(_lib.lib().cbb_backproject_device_band(
        vol_slab.data_ptr(), C.byref(g), int(z_begin), int(z_end),
        packed.data_ptr() + int(first) * nbb, int(width), int(height), int(count), _ptr(m),
        C.byref(band.c()), C.byref(oc), err, C.c_void_p(s.cuda_stream)))


def tma_plan(geometry: VolumeGeometry, width: int, height: int, z_begin: int, z_end: int,
             matrices: np.ndarray) -> dict:
    """cbb_tma_plan: whether the TMA-staged kernel runs for this slab and
    stack (one GPU), with its box size and ring depth. Host-only."""
    m = validate_matrices(matrices)
    out = _lib.TmaPlanC()
    _lib.check(_lib.lib().cbb_tma_plan(C.byref(geometry_c(geometry)), int(width), int(height),
                                       int(z_begin), int(z_end), _ptr(m), m.shape[0],
                                       C.byref(out)))
    return {k: int(getattr(out, k)) for k, _ in out._fields_}


def scan_device(raw, flags, err_flag=None, stream=None) -> None:
    """cbb_scan_device: per-projection numerator-range flags (uint32 / int32
    CUDA tensor of N entries) and the non-finite check (err_flag bit 2) of raw
    projections (contiguous CUDA float32 (N, rows, W))."""
    import torch

    stride = _rows_view_stride(raw, "scan_device")
    n, rows, w = raw.shape
    if flags.numel() * flags.element_size() < 4 * n:
        raise ValidationError("scan_device: flags too small")
    s = stream if stream is not None else torch.cuda.current_stream(raw.device)
    err = None if err_flag is None else err_flag.data_ptr()
    _lib.check(_lib.lib().cbb_scan_device(raw.data_ptr(), stride, w, rows, n, flags.data_ptr(),
                                          err, C.c_void_p(s.cuda_stream)))


def _rows_view_stride(raw, what: str) -> int:
    """(N, rows, W) CUDA float32 tensor whose rows are contiguous (a whole
    stack, or a band of rows of one: raw[:, r0:r0 + rn]); returns the
    projection stride in floats."""
    import torch

    if not (raw.is_cuda and raw.dtype == torch.float32 and raw.dim() == 3):
        raise ValidationError(f"{what}: raw must be a CUDA float32 (N, R, W) tensor")
    n, rows, w = raw.shape
    if raw.stride(2) != 1 or (rows > 1 and raw.stride(1) != w) or (n > 1 and raw.stride(0) < rows * w):
        raise ValidationError(f"{what}: raw rows must be contiguous (a stack or a band of one)")
    return int(raw.stride(0)) if n > 1 else rows * w


def backproject_raw_device(vol_slab, geometry: VolumeGeometry, z_begin: int, z_end: int, raw,
                           width: int, height: int, count: int, matrices: np.ndarray, flags,
                           options: Optional[Options] = None, err_flag=None, stream=None,
                           first: int = 0, band: Optional[RowBand] = None) -> None:
    """cbb_backproject_raw_device: back-projection straight from raw
    projections (CUDA float32 (N, rows, W) with contiguous rows: the full
    detector, or the band's rows with `band` -- e.g. raw[:, r0:r0 + rn] of a
    full stack), each block's footprint staged in shared memory by TMA;
    `flags` from scan_device over the same projections. Projections
    [first, first + count) of the tensor are used."""
    import torch

    if not (vol_slab.is_cuda and vol_slab.dtype == torch.float32 and vol_slab.is_contiguous()):
        raise ValidationError("backproject_raw_device: vol_slab must be a contiguous CUDA float32 tensor")
    stride = _rows_view_stride(raw, "backproject_raw_device")
    L = geometry.edge_voxels
    if vol_slab.numel() < (z_end - z_begin) * L * L:
        raise ValidationError("backproject_raw_device: slab tensor too small")
    m = validate_matrices(matrices)
    n, rows, w = raw.shape
    if m.shape[0] < count or first + count > n or w != width:
        raise ValidationError("backproject_raw_device: projection count or width mismatch")
    oc, _keep = (options or Options()).to_c()
    g = geometry_c(geometry)
    s = stream if stream is not None else torch.cuda.current_stream(vol_slab.device)
    err = None if err_flag is None else err_flag.data_ptr()
    _lib.check(_lib.lib().cbb_backproject_raw_device(
        vol_slab.data_ptr(), C.byref(g), int(z_begin), int(z_end),
        raw.data_ptr() + 4 * int(first) * stride, stride, int(width), int(height),
        None if band is None else C.byref(band.c()), int(count), _ptr(m),
        flags.data_ptr() + 4 * int(first), C.byref(oc), err, C.c_void_p(s.cuda_stream)))


def ramp_filter_device(raw, out, pixel_mm: float, stream=None) -> None:
    """FDK row-wise Shepp-Logan ramp filter on the GPU (cbb_ramp_filter_device):
    raw, out: contiguous CUDA float32 tensors (N, H, W) (may be the same)."""
    import torch

    for t in (raw, out):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.dim() == 3):
            raise ValidationError("ramp_filter_device: contiguous CUDA float32 (N, H, W) tensors")
    if raw.shape != out.shape:
        raise ValidationError("ramp_filter_device: shapes differ")
    n, h, w = raw.shape
    s = stream if stream is not None else torch.cuda.current_stream(raw.device)
    _lib.check(_lib.lib().cbb_ramp_filter_device(raw.data_ptr(), out.data_ptr(), w, h, n,
                                                 float(pixel_mm), C.c_void_p(s.cuda_stream)))


def compare_volumes_device(test, ref, denom_floor: float = 1e-6, stream=None) -> dict:
    """quality_metrics / max_relative_error of the reference harness
    (proj/src/bench.cpp:65-102) plus relL2, max|d|/range and the count of
    bitwise-different voxels, computed on the GPU (cbb_compare_volumes_device)."""
    import torch

    for t in (test, ref):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValidationError("compare_volumes_device: contiguous CUDA float32 tensors")
    if test.numel() != ref.numel() or test.numel() == 0:
        raise ValidationError("compare_volumes_device: sizes differ or empty")
    s = stream if stream is not None else torch.cuda.current_stream(test.device)
    out = _lib.VolumeDiffC()
    _lib.check(_lib.lib().cbb_compare_volumes_device(test.data_ptr(), ref.data_ptr(),
                                                     test.numel(), float(denom_floor),
                                                     C.byref(out), C.c_void_p(s.cuda_stream)))
    return out.to_dict()


def backproject_texture_device(vol_slab, geometry: VolumeGeometry, z_begin: int, z_end: int,
                               raw, matrices: np.ndarray, stream=None) -> None:
    """Side variant: hardware-texture bilinear back-projection of raw CUDA
    float32 projections (N, H, W) -- NOT parity-exact (8-bit texture weights,
    floor addressing, FMA coordinates); reported only as a side number."""
    import torch

    if not (raw.is_cuda and raw.dtype == torch.float32 and raw.is_contiguous() and raw.dim() == 3):
        raise ValidationError("backproject_texture_device: raw must be CUDA float32 (N, H, W)")
    m = validate_matrices(matrices)
    n, h, w = raw.shape
    g = geometry_c(geometry)
    s = stream if stream is not None else torch.cuda.current_stream(raw.device)
    _lib.check(_lib.lib().cbb_backproject_texture_device(
        vol_slab.data_ptr(), C.byref(g), int(z_begin), int(z_end), raw.data_ptr(), w, h, n,
        _ptr(m), C.c_void_p(s.cuda_stream)))


def launch_count() -> int:
    return int(_lib.lib().cbb_launch_count())


def device_count() -> int:
    return int(_lib.lib().cbb_device_count())

"""ctypes binding of libconebeam_b200.so (declared in include/conebeam_b200.h).

The product path has no fallback: if the library is missing or cannot be
loaded, ``lib()`` raises. Nothing here imports the oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import InternalError, error_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libconebeam_b200.so")
# experiments only: load another build of the same library (e.g. a kernel
# variant compiled with different -D flags); the product default is LIB_PATH
LIB_PATH = os.environ.get("CBB_LIB_PATH", LIB_PATH)

# Every symbol declared in include/conebeam_b200.h (checked by tests).
EXPORTS = (
    "cbb_status_name", "cbb_last_error", "cbb_version", "cbb_device_count",
    "cbb_options_defaults", "cbb_backproject", "cbb_reconstruct",
    "cbb_session_create", "cbb_session_backproject", "cbb_session_finish",
    "cbb_session_free", "cbb_packed_layout", "cbb_pack_device",
    "cbb_backproject_device", "cbb_launch_count", "cbb_ramp_filter_device",
    "cbb_compare_volumes_device", "cbb_stack_file_query", "cbb_reconstruct_file",
    "cbb_backproject_texture_device", "cbb_row_band_for_slab", "cbb_pack_device_band",
    "cbb_backproject_device_band", "cbb_check_finite_device", "cbb_reconstruct_images",
    "cbb_release_cached_memory", "cbb_ipc_alloc", "cbb_ipc_free", "cbb_ipc_open",
    "cbb_ipc_close", "cbb_stream_write_flag", "cbb_stream_wait_flag", "cbb_memcpy_h2d_async",
    "cbb_scan_device", "cbb_backproject_raw_device", "cbb_tma_plan",
)


class RowBandC(C.Structure):
    _fields_ = [("raw_row0", C.c_int32), ("raw_rows", C.c_int32),
                ("cell_row0", C.c_int32), ("cell_rows", C.c_int32)]


class StackFileInfoC(C.Structure):
    _fields_ = [("edge_voxels", C.c_int32), ("voxel_mm", C.c_double), ("origin_mm", C.c_double),
                ("count", C.c_int32), ("width", C.c_int32), ("height", C.c_int32)]


class VolumeGeometryC(C.Structure):
    _fields_ = [("edge_voxels", C.c_int32), ("voxel_mm", C.c_double),
                ("origin_mm", C.c_double)]


class OptionsC(C.Structure):
    _fields_ = [("num_gpus", C.c_int32), ("device_ids", C.POINTER(C.c_int32)),
                ("batch", C.c_int32), ("mode", C.c_int32), ("cull", C.c_int32),
                ("volume_is_zero", C.c_int32), ("slab_begin", C.c_int32),
                ("slab_end", C.c_int32), ("ramp_filter", C.c_int32),
                ("filter_pixel_mm", C.c_double), ("count_culled", C.c_int32)]


class TmaPlanC(C.Structure):
    _fields_ = [("staged", C.c_int32), ("box_width", C.c_int32), ("box_rows", C.c_int32),
                ("stages", C.c_int32), ("footprint_width", C.c_int32),
                ("footprint_rows", C.c_int32)]


class RunStatsC(C.Structure):
    _fields_ = [("total_seconds", C.c_double), ("h2d_seconds", C.c_double),
                ("kernel_seconds", C.c_double), ("d2h_seconds", C.c_double),
                ("voxel_updates", C.c_uint64), ("guarded_batches", C.c_uint64),
                ("num_gpus", C.c_int32), ("per_gpu_kernel_seconds", C.c_double * 8),
                ("culled_updates", C.c_uint64), ("culled_fraction", C.c_double)]

    def to_dict(self) -> dict:
        return {
            "total_seconds": self.total_seconds, "h2d_seconds": self.h2d_seconds,
            "kernel_seconds": self.kernel_seconds, "d2h_seconds": self.d2h_seconds,
            "voxel_updates": int(self.voxel_updates),
            "guarded_batches": int(self.guarded_batches), "num_gpus": int(self.num_gpus),
            "per_gpu_kernel_seconds": list(self.per_gpu_kernel_seconds)[: max(self.num_gpus, 0)],
            "culled_updates": int(self.culled_updates),
            "culled_fraction": self.culled_fraction,
        }


class VolumeDiffC(C.Structure):
    _fields_ = [("mse", C.c_double), ("psnr_db", C.c_double),
                ("max_relative_error", C.c_double), ("rel_l2", C.c_double),
                ("max_abs", C.c_double), ("ref_min", C.c_double), ("ref_max", C.c_double),
                ("max_abs_over_range", C.c_double), ("bitwise_different", C.c_uint64)]

    def to_dict(self) -> dict:
        return {k: (int(getattr(self, k)) if k == "bitwise_different" else getattr(self, k))
                for k, _ in self._fields_}


_lock = threading.Lock()
_lib = None

_FP = C.POINTER(C.c_float)
_DP = C.POINTER(C.c_double)
_VP = C.c_void_p


def _declare(L) -> None:
    L.cbb_status_name.restype = C.c_char_p
    L.cbb_status_name.argtypes = [C.c_int]
    L.cbb_last_error.restype = C.c_char_p
    L.cbb_last_error.argtypes = []
    L.cbb_version.restype = C.c_char_p
    L.cbb_device_count.restype = C.c_int32
    L.cbb_options_defaults.restype = None
    L.cbb_options_defaults.argtypes = [C.POINTER(OptionsC)]
    L.cbb_backproject.restype = C.c_int
    L.cbb_backproject.argtypes = [_VP, C.POINTER(VolumeGeometryC), _VP, C.c_int32, C.c_int32, _VP]
    L.cbb_reconstruct.restype = C.c_int
    L.cbb_reconstruct.argtypes = [_VP, C.POINTER(VolumeGeometryC), _VP, C.c_int32, C.c_int32,
                                  C.c_int32, _VP, C.POINTER(OptionsC), C.POINTER(RunStatsC)]
    L.cbb_reconstruct_images.restype = C.c_int
    L.cbb_reconstruct_images.argtypes = [_VP, C.POINTER(VolumeGeometryC), _VP, C.c_int32,
                                         C.c_int32, C.c_int32, _VP, C.POINTER(OptionsC),
                                         C.POINTER(RunStatsC)]
    L.cbb_session_create.restype = C.c_int
    L.cbb_session_create.argtypes = [C.POINTER(VolumeGeometryC), C.c_int32, C.c_int32, _VP,
                                     C.POINTER(OptionsC), C.POINTER(_VP)]
    L.cbb_session_backproject.restype = C.c_int
    L.cbb_session_backproject.argtypes = [_VP, _VP, _VP]
    L.cbb_session_finish.restype = C.c_int
    L.cbb_session_finish.argtypes = [_VP, _VP, C.POINTER(RunStatsC)]
    L.cbb_session_free.restype = None
    L.cbb_session_free.argtypes = [_VP]
    L.cbb_packed_layout.restype = C.c_int
    L.cbb_packed_layout.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
    L.cbb_pack_device.restype = C.c_int
    L.cbb_pack_device.argtypes = [_VP, C.c_int32, C.c_int32, C.c_int32, _VP, _VP]
    L.cbb_backproject_device.restype = C.c_int
    L.cbb_backproject_device.argtypes = [_VP, C.POINTER(VolumeGeometryC), C.c_int32, C.c_int32,
                                         _VP, C.c_int32, C.c_int32, C.c_int32, _VP,
                                         C.POINTER(OptionsC), _VP, _VP]
    L.cbb_ramp_filter_device.restype = C.c_int
    L.cbb_ramp_filter_device.argtypes = [_VP, _VP, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                         _VP]
    L.cbb_backproject_texture_device.restype = C.c_int
    L.cbb_backproject_texture_device.argtypes = [_VP, C.POINTER(VolumeGeometryC), C.c_int32,
                                                 C.c_int32, _VP, C.c_int32, C.c_int32,
                                                 C.c_int32, _VP, _VP]
    L.cbb_stack_file_query.restype = C.c_int
    L.cbb_stack_file_query.argtypes = [C.c_char_p, C.POINTER(StackFileInfoC)]
    L.cbb_reconstruct_file.restype = C.c_int
    L.cbb_reconstruct_file.argtypes = [_VP, C.c_char_p, C.POINTER(OptionsC),
                                       C.POINTER(RunStatsC)]
    L.cbb_compare_volumes_device.restype = C.c_int
    L.cbb_compare_volumes_device.argtypes = [_VP, _VP, C.c_int64, C.c_double,
                                             C.POINTER(VolumeDiffC), _VP]
    L.cbb_row_band_for_slab.restype = C.c_int
    L.cbb_row_band_for_slab.argtypes = [C.POINTER(VolumeGeometryC), C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, _VP, C.c_int32,
                                        C.POINTER(RowBandC)]
    L.cbb_pack_device_band.restype = C.c_int
    L.cbb_pack_device_band.argtypes = [_VP, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(RowBandC), _VP, _VP, _VP]
    L.cbb_backproject_device_band.restype = C.c_int
    L.cbb_backproject_device_band.argtypes = [_VP, C.POINTER(VolumeGeometryC), C.c_int32,
                                              C.c_int32, _VP, C.c_int32, C.c_int32, C.c_int32,
                                              _VP, C.POINTER(RowBandC), C.POINTER(OptionsC),
                                              _VP, _VP]
    L.cbb_check_finite_device.restype = C.c_int
    L.cbb_check_finite_device.argtypes = [_VP, C.c_int64, _VP, _VP]
    L.cbb_tma_plan.restype = C.c_int
    L.cbb_tma_plan.argtypes = [C.POINTER(VolumeGeometryC), C.c_int32, C.c_int32, C.c_int32,
                               C.c_int32, _VP, C.c_int32, C.POINTER(TmaPlanC)]
    L.cbb_scan_device.restype = C.c_int
    L.cbb_scan_device.argtypes = [_VP, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _VP, _VP,
                                  _VP]
    L.cbb_backproject_raw_device.restype = C.c_int
    L.cbb_backproject_raw_device.argtypes = [_VP, C.POINTER(VolumeGeometryC), C.c_int32,
                                             C.c_int32, _VP, C.c_int64, C.c_int32, C.c_int32,
                                             C.POINTER(RowBandC), C.c_int32, _VP, _VP,
                                             C.POINTER(OptionsC), _VP, _VP]
    for name, args in (("cbb_ipc_alloc", [C.c_int64, C.POINTER(_VP), _VP]),
                       ("cbb_ipc_free", [_VP]), ("cbb_ipc_open", [_VP, C.POINTER(_VP)]),
                       ("cbb_ipc_close", [_VP]),
                       ("cbb_stream_write_flag", [_VP, C.c_uint32, _VP]),
                       ("cbb_stream_wait_flag", [_VP, C.c_uint32, _VP]),
                       ("cbb_memcpy_h2d_async", [_VP, _VP, C.c_int64, _VP])):
        fn = getattr(L, name)
        fn.restype = C.c_int
        fn.argtypes = args
    L.cbb_release_cached_memory.restype = C.c_int
    L.cbb_release_cached_memory.argtypes = []
    L.cbb_launch_count.restype = C.c_uint64
    L.cbb_launch_count.argtypes = []


def lib():
    """Loads libconebeam_b200.so once; raises InternalError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise InternalError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(make -C paper_1401_3615_b200/csrc); there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            _declare(L)
            _lib = L
    return _lib


def check(status: int) -> None:
    """Raises the exception matching a non-zero cbb_status with cbb_last_error()."""
    if status != 0:
        msg = lib().cbb_last_error().decode(errors="replace")
        raise error_for_status(status, msg)

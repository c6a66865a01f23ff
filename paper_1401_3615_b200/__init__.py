"""paper_1401_3615_b200 -- B200-native voxel-driven FDK back-projection.

Drop-in for the reference's hot path (proj/src/kernel_ref.cpp:5-38,
proj/src/kernel_opt.cpp:658-716) through the C ABI in include/conebeam_b200.h.
"""
from .backproject import (MODE_EXACT, MODE_FAST, Options, RowBand, Session, backproject,
                          backproject_device, backproject_texture_device, check_finite_device,
                          compare_volumes_device,
                          device_count, launch_count, pack_device, pack_device_band,
                          packed_layout, ramp_filter_device, reconstruct, reconstruct_arrays,
                          backproject_raw_device, scan_device, tma_plan,
                          reconstruct_file, reconstruct_images, release_cached_memory,
                          row_band_for_slab,
                          stack_file_info)
from .dataset import ProjectionStack, Volume, read_stack, read_volume, write_stack, write_volume
from .errors import (ConebeamError, FormatError, GeometryError, InternalError, IOError_,
                     OutOfMemoryError, TruncatedError, ValidationError)
from .geometry import (TrajectoryConfig, VolumeGeometry, dehomogenize, forward_project,
                       make_circular_trajectory, world_from_voxel)

__all__ = [
    "MODE_EXACT", "MODE_FAST", "Options", "RowBand", "Session", "backproject",
    "backproject_device", "backproject_texture_device", "check_finite_device", "compare_volumes_device",
    "pack_device_band", "release_cached_memory", "row_band_for_slab",
    "backproject_raw_device", "scan_device", "tma_plan",
    "device_count", "launch_count", "pack_device", "packed_layout", "ramp_filter_device", "reconstruct",
    "reconstruct_arrays", "reconstruct_file", "reconstruct_images", "stack_file_info", "ProjectionStack", "Volume", "read_stack", "read_volume",
    "write_stack", "write_volume", "ConebeamError", "FormatError", "GeometryError",
    "InternalError", "IOError_", "OutOfMemoryError", "TruncatedError", "ValidationError",
    "TrajectoryConfig", "VolumeGeometry", "dehomogenize", "forward_project",
    "make_circular_trajectory", "world_from_voxel",
]

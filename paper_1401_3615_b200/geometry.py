"""Geometry conventions of the reference, restated for the host side.

Mirrors proj/include/conebeam/geometry.hpp and proj/src/geometry.cpp:
  * VolumeGeometry (geometry.hpp:15-34): voxel index i -> origin + i * voxel_mm;
    ``centered`` puts the volume centre on the world origin (geometry.cpp:26-33).
  * Projection matrices are 12 doubles, column-major 3x4 (geometry.hpp:47-65):
        u = wx*a0 + wy*a3 + wz*a6 + a9
        v = wx*a1 + wy*a4 + wz*a7 + a10
        w = wx*a2 + wy*a5 + wz*a8 + a11
    normalised so that w(isocenter) == 1.
  * make_circular_trajectory (geometry.cpp:79-116).
Matrices are numpy float64 arrays of shape (N, 12).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import GeometryError, ValidationError


@dataclass(frozen=True)
class VolumeGeometry:
    edge_voxels: int
    voxel_mm: float = 1.0
    origin_mm: float = 0.0

    def validate(self) -> None:
        """VolumeGeometry::validate (proj/src/geometry.cpp:17-24)."""
        if self.edge_voxels < 1:
            raise ValidationError("VolumeGeometry: field 'edge_voxels' must be >= 1")
        if not (self.voxel_mm > 0.0) or not math.isfinite(self.voxel_mm):
            raise ValidationError("VolumeGeometry: field 'voxel_mm' must be positive and finite")
        if not math.isfinite(self.origin_mm):
            raise ValidationError("VolumeGeometry: field 'origin_mm' must be finite")

    @property
    def voxel_count(self) -> int:
        return self.edge_voxels ** 3

    @staticmethod
    def centered(edge_voxels: int, voxel_mm: float) -> "VolumeGeometry":
        """origin = -(L-1)/2 * voxel size (proj/src/geometry.cpp:26-33)."""
        g = VolumeGeometry(int(edge_voxels), float(voxel_mm),
                           -0.5 * float(edge_voxels - 1) * float(voxel_mm))
        g.validate()
        return g


@dataclass
class TrajectoryConfig:
    """proj/include/conebeam/geometry.hpp:67-83."""

    num_projections: int
    source_isocenter_mm: float
    source_detector_mm: float
    detector_width: int
    detector_height: int
    pixel_size_mm: float
    angular_range_rad: float = 2.0 * math.pi

    def validate(self) -> None:
        """TrajectoryConfig::validate (proj/src/geometry.cpp:41-58)."""
        if self.num_projections < 1:
            raise ValidationError("TrajectoryConfig: field 'num_projections' must be >= 1")
        for name in ("source_isocenter_mm", "source_detector_mm", "pixel_size_mm",
                     "angular_range_rad"):
            val = getattr(self, name)
            if not (val > 0.0) or not math.isfinite(val):
                raise ValidationError(f"TrajectoryConfig: field '{name}' must be positive and finite")
        if self.source_detector_mm <= self.source_isocenter_mm:
            raise ValidationError(
                "TrajectoryConfig: field 'source_detector_mm' must exceed source_isocenter_mm")
        if self.detector_width < 1:
            raise ValidationError("TrajectoryConfig: field 'detector_width' must be >= 1")
        if self.detector_height < 1:
            raise ValidationError("TrajectoryConfig: field 'detector_height' must be >= 1")


def world_from_voxel(g: VolumeGeometry, x: int, y: int, z: int):
    """proj/src/geometry.cpp:60-64 (double precision)."""
    return (g.origin_mm + x * g.voxel_mm, g.origin_mm + y * g.voxel_mm,
            g.origin_mm + z * g.voxel_mm)


def forward_project(a, wx: float, wy: float, wz: float):
    """(u, v, w) of a world point, double precision (proj/src/geometry.cpp:66-71)."""
    return (wx * a[0] + wy * a[3] + wz * a[6] + a[9],
            wx * a[1] + wy * a[4] + wz * a[7] + a[10],
            wx * a[2] + wy * a[5] + wz * a[8] + a[11])


def dehomogenize(u: float, v: float, w: float):
    """(u/w, v/w); w == 0 raises GeometryError (proj/src/geometry.cpp:73-77)."""
    if w == 0.0:
        raise GeometryError("dehomogenize: w == 0, ray parallel to the detector plane")
    return (u / w, v / w)


def make_circular_trajectory(c: TrajectoryConfig) -> np.ndarray:
    """One matrix per angle, angle_i = range * i / N (proj/src/geometry.cpp:79-116).

    Source at R(cos, sin, 0); detector axes e_u = (-sin, cos, 0), e_v = (0, 0, 1);
    rows scaled by 1/R so that w(0,0,0) == 1; the isocentre projects to
    ((W-1)/2, (H-1)/2).
    """
    c.validate()
    radius = float(c.source_isocenter_mm)
    focal_px = c.source_detector_mm / c.pixel_size_mm
    cu = 0.5 * float(c.detector_width - 1)
    cv = 0.5 * float(c.detector_height - 1)
    out = np.zeros((c.num_projections, 12), dtype=np.float64)
    for i in range(c.num_projections):
        angle = c.angular_range_rad * float(i) / float(c.num_projections)
        cs = math.cos(angle)
        sn = math.sin(angle)
        a = out[i]
        a[0] = (-focal_px * sn - cu * cs) / radius
        a[3] = (focal_px * cs - cu * sn) / radius
        a[6] = 0.0
        a[9] = cu
        a[1] = (-cv * cs) / radius
        a[4] = (-cv * sn) / radius
        a[7] = focal_px / radius
        a[10] = cv
        a[2] = -cs / radius
        a[5] = -sn / radius
        a[8] = 0.0
        a[11] = 1.0
    return out


def validate_matrices(mats: np.ndarray) -> np.ndarray:
    """ProjectionMatrix::validate (proj/src/geometry.cpp:35-39) over an (N,12) array."""
    m = np.ascontiguousarray(mats, dtype=np.float64)
    if m.ndim == 1:
        m = m.reshape(1, 12)
    if m.ndim != 2 or m.shape[1] != 12:
        raise ValidationError("ProjectionMatrix: expected shape (N, 12)")
    bad = ~np.isfinite(m)
    if bad.any():
        i = int(np.argwhere(bad)[0][1])
        raise ValidationError(f"ProjectionMatrix: field 'a[{i}]' must be finite")
    return m

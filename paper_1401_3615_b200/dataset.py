"""Host data types and file formats, mirroring proj/include/conebeam/dataset.hpp.

  * Volume: float32 voxels, linear index (z*L + y)*L + x (dataset.hpp:39-57);
    held here as a C-contiguous numpy array of shape (L, L, L) indexed [z, y, x].
  * ProjectionStack: geometry + N matrices (N, 12) float64 + N images
    (N, H, W) float32, row-major iy*W + ix (dataset.hpp:15-37).
  * CBPS stack / CBPV volume little-endian files (dataset.hpp:62-72,
    proj/src/dataset.cpp:155-246), byte-compatible with the reference.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from .errors import FormatError, GeometryError, IOError_, TruncatedError, ValidationError
from .geometry import VolumeGeometry, validate_matrices

_STACK_MAGIC = b"CBPS"
_VOLUME_MAGIC = b"CBPV"
_VERSION = 1


def _require_finite(a: np.ndarray, what: str) -> None:
    if not np.isfinite(a).all():
        raise ValidationError(f"{what} contains non-finite values")


@dataclass
class Volume:
    geometry: VolumeGeometry
    voxels: np.ndarray = field(default=None)  # (L, L, L) float32, [z, y, x]

    def __post_init__(self):
        self.geometry.validate()
        L = self.geometry.edge_voxels
        if self.voxels is None:
            self.voxels = np.zeros((L, L, L), dtype=np.float32)
        else:
            self.voxels = np.ascontiguousarray(self.voxels, dtype=np.float32).reshape(L, L, L)

    def at(self, x: int, y: int, z: int) -> float:
        return float(self.voxels[z, y, x])

    def validate(self) -> None:
        """Volume::validate (proj/src/dataset.cpp:146-151)."""
        self.geometry.validate()
        L = self.geometry.edge_voxels
        if self.voxels.shape != (L, L, L):
            raise ValidationError("Volume: voxel buffer length != L^3")
        _require_finite(self.voxels, "Volume")


@dataclass
class ProjectionStack:
    geometry: VolumeGeometry
    matrices: np.ndarray  # (N, 12) float64
    images: np.ndarray    # (N, H, W) float32

    def __post_init__(self):
        self.matrices = validate_matrices(self.matrices)
        self.images = np.ascontiguousarray(self.images, dtype=np.float32)
        if self.images.ndim == 2:
            self.images = self.images[None]

    @property
    def count(self) -> int:
        return int(self.images.shape[0])

    @property
    def width(self) -> int:
        return int(self.images.shape[2])

    @property
    def height(self) -> int:
        return int(self.images.shape[1])

    def validate(self, check_finite: bool = True) -> None:
        """ProjectionStack::validate (proj/src/dataset.cpp:131-144)."""
        self.geometry.validate()
        if self.images.ndim != 3 or self.count < 1:
            raise ValidationError("ProjectionStack: at least one projection required")
        if self.matrices.shape[0] != self.count:
            raise ValidationError("ProjectionStack: images and matrices differ in length")
        if self.width < 1 or self.height < 1:
            raise ValidationError("ProjectionImage: dimensions must be >= 1")
        if check_finite:
            _require_finite(self.images, "ProjectionImage")


def check_same_geometry(vol: Volume, stack: ProjectionStack, who: str) -> None:
    if vol.geometry != stack.geometry:
        raise GeometryError(f"{who}: volume and stack geometries differ")


# --- file formats -------------------------------------------------------------

def write_stack(path: str, s: ProjectionStack) -> None:
    """CBPS writer (proj/src/dataset.cpp:155-179)."""
    s.validate()
    try:
        with open(path, "wb") as f:
            f.write(_STACK_MAGIC)
            f.write(struct.pack("<HHIII", _VERSION, 0, s.width, s.height, s.count))
            g = s.geometry
            f.write(struct.pack("<ddI", g.voxel_mm, g.origin_mm, g.edge_voxels))
            mats = s.matrices.astype("<f8")
            imgs = s.images.astype("<f4")
            for i in range(s.count):
                f.write(mats[i].tobytes())
                f.write(imgs[i].tobytes())
    except OSError as e:
        raise IOError_(f"cannot open '{path}' for writing: {e}") from e


def _read_exact(f, n: int, what: str) -> bytes:
    b = f.read(n)
    if len(b) != n:
        raise TruncatedError(f"file ends inside {what}")
    return b


def _check_magic(f, magic: bytes, kind: str) -> None:
    if _read_exact(f, 4, "magic") != magic:
        raise FormatError(f"not a {kind} file (magic mismatch)")
    version, _ = struct.unpack("<HH", _read_exact(f, 4, "version"))
    if version != _VERSION:
        raise FormatError(f"{kind} file version {version} not supported (expected {_VERSION})")


def read_stack(path: str) -> ProjectionStack:
    """CBPS reader (proj/src/dataset.cpp:181-212)."""
    try:
        f = open(path, "rb")
    except OSError as e:
        raise IOError_(f"cannot open '{path}' for reading") from e
    with f:
        _check_magic(f, _STACK_MAGIC, "stack")
        width, height, count = struct.unpack("<III", _read_exact(f, 12, "header"))
        voxel_mm, origin_mm, L = struct.unpack("<ddI", _read_exact(f, 20, "header"))
        if width < 1 or height < 1 or count < 1:
            raise FormatError("stack header has zero width, height, or count")
        g = VolumeGeometry(int(L), voxel_mm, origin_mm)
        g.validate()
        rec = 96 + 4 * width * height
        payload = f.read(rec * count)
        if len(payload) != rec * count:
            raise TruncatedError("file ends inside projection intensities")
        if f.read(1):
            raise FormatError("stack file has trailing bytes after payload")
    buf = np.frombuffer(payload, dtype=np.uint8).reshape(count, rec)
    mats = buf[:, :96].copy().view("<f8").astype(np.float64).reshape(count, 12)
    imgs = buf[:, 96:].copy().view("<f4").astype(np.float32).reshape(count, height, width)
    s = ProjectionStack(g, mats, imgs)
    s.validate()
    return s


def write_volume(path: str, v: Volume) -> None:
    """CBPV writer (proj/src/dataset.cpp:216-229)."""
    v.validate()
    try:
        with open(path, "wb") as f:
            f.write(_VOLUME_MAGIC)
            g = v.geometry
            f.write(struct.pack("<HHIdd", _VERSION, 0, g.edge_voxels, g.voxel_mm, g.origin_mm))
            f.write(v.voxels.astype("<f4").tobytes())
    except OSError as e:
        raise IOError_(f"cannot open '{path}' for writing: {e}") from e


def read_volume(path: str) -> Volume:
    """CBPV reader (proj/src/dataset.cpp:231-246)."""
    try:
        f = open(path, "rb")
    except OSError as e:
        raise IOError_(f"cannot open '{path}' for reading") from e
    with f:
        _check_magic(f, _VOLUME_MAGIC, "volume")
        L, voxel_mm, origin_mm = struct.unpack("<Idd", _read_exact(f, 20, "header"))
        g = VolumeGeometry(int(L), voxel_mm, origin_mm)
        g.validate()
        n = 4 * L ** 3
        payload = f.read(n)
        if len(payload) != n:
            raise TruncatedError("file ends inside voxel payload")
        if f.read(1):
            raise FormatError("volume file has trailing bytes after payload")
    v = Volume(g, np.frombuffer(payload, dtype="<f4").astype(np.float32).reshape(L, L, L))
    v.validate()
    return v


def stack_file_bytes(width: int, height: int, count: int) -> int:
    return 4 + 2 + 2 + 12 + 20 + count * (96 + 4 * width * height)


__all__ = ["Volume", "ProjectionStack", "write_stack", "read_stack", "write_volume",
           "read_volume", "check_same_geometry", "stack_file_bytes"]

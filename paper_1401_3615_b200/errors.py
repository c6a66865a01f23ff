"""Error hierarchy mirroring the reference (proj/include/conebeam/errors.hpp:10-44)
and its C status mapping (proj/include/conebeam/capi.h:20-29)."""


class ConebeamError(RuntimeError):
    """Base class of all library errors (conebeam::error)."""

    status = 7


class ValidationError(ConebeamError):
    """Invalid arguments or configuration (conebeam::validation_error)."""

    status = 1


class IOError_(ConebeamError):
    """Failure to open, read, or write a file (conebeam::io_error)."""

    status = 2


class FormatError(ConebeamError):
    """Readable file in the wrong format (conebeam::format_error)."""

    status = 3


class TruncatedError(FormatError):
    """Payload shorter than the header promises (conebeam::truncated_error)."""

    status = 4


class GeometryError(ConebeamError):
    """Degenerate projection geometry, e.g. a voxel with w == 0 (conebeam::geometry_error)."""

    status = 5


class OutOfMemoryError(ConebeamError):
    """Host or device allocation failure (CB_ERR_NOMEM)."""

    status = 6


class InternalError(ConebeamError):
    """CUDA failure or missing device (CB_ERR_INTERNAL)."""

    status = 7


_BY_STATUS = {
    1: ValidationError,
    2: IOError_,
    3: FormatError,
    4: TruncatedError,
    5: GeometryError,
    6: OutOfMemoryError,
    7: InternalError,
}


def error_for_status(status: int, message: str) -> ConebeamError:
    """Maps a cbb_status / cb_status value to the matching exception."""
    return _BY_STATUS.get(int(status), InternalError)(message)

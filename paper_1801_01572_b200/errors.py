"""Exception hierarchy of the reference (proj/include/loopkit/errors.hpp:9-74).

lk_status codes returned by the C ABI map back onto these classes so callers
of the Python mirror catch the same types the reference's callers catch.
"""
from __future__ import annotations

from . import abi


class Error(RuntimeError):
    """Base class for all library errors (errors.hpp:9-11)."""


class EmptyCloud(Error):
    pass


class RotationTooLarge(Error):
    pass


class DegenerateConfiguration(Error):
    pass


class TooFewPoints(Error):
    pass


class MissingNormals(Error):
    pass


class MissingData(Error):
    pass


class NoCorrespondences(Error):
    pass


class SingularSystem(Error):
    pass


class ParseError(Error):
    """A malformed input file; the message is "path:line: what" (errors.hpp:64-69)."""


class CudaError(Error):
    """A CUDA failure on the device path (no CPU fallback exists)."""


class NcclError(Error):
    pass


_BY_STATUS = {
    abi.LK_EMPTY_CLOUD: EmptyCloud,
    abi.LK_TOO_FEW_POINTS: TooFewPoints,
    abi.LK_MISSING_DATA: MissingData,
    abi.LK_MISSING_NORMALS: MissingNormals,
    abi.LK_NO_CORRESPONDENCES: NoCorrespondences,
    abi.LK_DEGENERATE: DegenerateConfiguration,
    abi.LK_INVALID_ARGUMENT: Error,
    abi.LK_CUDA_ERROR: CudaError,
    abi.LK_NCCL_ERROR: NcclError,
    abi.LK_ROTATION_TOO_LARGE: RotationTooLarge,
    abi.LK_INTERNAL_ERROR: Error,
}


def check(status: int, allow=(abi.LK_OK,)) -> int:
    """Raise the reference exception type for a failing lk_status."""
    if status in allow:
        return status
    cls = _BY_STATUS.get(status, Error)
    raise cls(abi.last_error() or f"lk_status {status}")

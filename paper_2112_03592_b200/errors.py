"""Exception taxonomy mirroring aprkit/errors.hpp:9-41.

C-ABI status codes (include/aprgpu.h) map back onto these types, exactly as the
C++ shim (include/aprkit_gpu.hpp) maps them onto aprkit's C++ exceptions.
"""
from __future__ import annotations


class RangeError(IndexError):
    """aprkit::RangeError (std::out_of_range): out-of-range levels, rows, extents."""


class IntegrityError(RuntimeError):
    """aprkit::IntegrityError: corrupt or inconsistent sparse structure."""


class CapabilityError(RuntimeError):
    """aprkit::CapabilityError: request exceeds a capability (extent > 13, y > 65536)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the device path."""


class NcclError(RuntimeError):
    """An NCCL failure in the multi-GPU path."""


class DeviceOutOfMemory(MemoryError):
    """Device allocation failure."""


class InvalidArgument(ValueError):
    """Bad argument at the C-ABI (null pointer, unknown enum, ...)."""


class IoError(RuntimeError):
    """aprkit::IoError: a file that cannot be opened, read or written."""


class BadFormatError(IoError):
    """aprkit::BadFormatError: malformed file content."""


class TruncatedFileError(IoError):
    """aprkit::TruncatedFileError: the stream ends early."""


_BY_STATUS = {
    1: RangeError,
    2: CapabilityError,
    3: IntegrityError,
    4: CudaError,
    5: NcclError,
    6: DeviceOutOfMemory,
    7: InvalidArgument,
    8: IoError,
    9: BadFormatError,
    10: TruncatedFileError,
}


def from_status(status: int, msg: str) -> Exception:
    return _BY_STATUS.get(status, RuntimeError)(msg)

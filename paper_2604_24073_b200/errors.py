"""Exception classes of the reference (proj/include/freescale/errors.hpp:9-31)
plus the std:: classes its hot path throws, keyed by the fsx.h status codes.

The C++ reference throws std::invalid_argument / std::domain_error /
std::out_of_range from the embedding and partition code; the Python mirror
raises InvalidArgument / DomainError / OutOfRange (ValueError / IndexError
subclasses) with the same message text.
"""


class FreeScaleError(RuntimeError):
    pass


class ConfigError(FreeScaleError):
    """errors.hpp:9-13"""


class CollectiveError(FreeScaleError):
    """errors.hpp:15-20"""


class ProtocolError(FreeScaleError):
    """errors.hpp:22-26"""


class IoError(FreeScaleError):
    """errors.hpp:28-31"""


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ValueError):
    """std::domain_error"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class CudaError(RuntimeError):
    """CUDA runtime/driver failure or allocation failure (no reference analogue)."""


_BY_CODE = {
    -1: InvalidArgument,
    -2: DomainError,
    -3: OutOfRange,
    -4: ProtocolError,
    -5: CollectiveError,
    -6: ConfigError,
    -7: CudaError,
    -8: CudaError,
    -9: IoError,
}


def from_status(code: int, msg: str) -> Exception:
    return _BY_CODE.get(code, CudaError)(msg)

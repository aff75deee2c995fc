"""Exception taxonomy of the reference (proj/include/svdkit/errors.hpp:11-55).

C-ABI status codes (include/svdk.h) map onto these one-to-one; engine-only
failures (CUDA, NCCL, allocation, bad state) derive from EngineError.
"""


class Error(RuntimeError):
    """Base class for all svdkit errors (errors.hpp:11-15)."""


class DimensionError(Error):
    """Shape mismatch between operands (errors.hpp:17-21)."""


class ParamError(Error):
    """A parameter is outside its documented domain (errors.hpp:23-27)."""


class NumericalError(Error):
    """An iterative kernel failed to reach its target (errors.hpp:29-39)."""

    def __init__(self, what: str, residual: float = 0.0):
        super().__init__(what)
        self._residual = float(residual)

    def residual(self) -> float:
        return self._residual


class FormatError(Error):
    """Malformed input bytes / text, with the byte offset or line (errors.hpp:40-49)."""

    def __init__(self, what: str, offset: int = 0):
        super().__init__(what)
        self._offset = int(offset)

    def offset(self) -> int:
        return self._offset


class IoError(Error):
    """File open / read / write failure (errors.hpp:51-55)."""


class EngineError(Error):
    """CUDA / NCCL / allocation failure inside the B200 engine (no reference analogue)."""


SVDK_OK, SVDK_E_DIM, SVDK_E_PARAM, SVDK_E_NUMERICAL = 0, 1, 2, 3
SVDK_E_CUDA, SVDK_E_NCCL, SVDK_E_NOMEM, SVDK_E_STATE = 4, 5, 6, 7
SVDK_E_FORMAT, SVDK_E_IO = 8, 9


def raise_for_status(code: int, message: str, residual: float = 0.0, offset: int = 0) -> None:
    if code == SVDK_OK:
        return
    if code == SVDK_E_DIM:
        raise DimensionError(message)
    if code == SVDK_E_PARAM:
        raise ParamError(message)
    if code == SVDK_E_NUMERICAL:
        raise NumericalError(message, residual)
    if code == SVDK_E_FORMAT:
        raise FormatError(message, offset)
    if code == SVDK_E_IO:
        raise IoError(message)
    raise EngineError(f"[svdk status {code}] {message}")

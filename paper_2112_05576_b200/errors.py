"""Exception classes mirroring proj/include/edgealign/errors.h:14-75.

The C-ABI returns an ea_status; `raise_for_status` maps it onto the class the
reference would have thrown, carrying the same message text.
"""
from . import abi


class Error(RuntimeError):
    """edgealign::Error  errors.h:14-17"""


class ParseError(Error):
    """errors.h:20-29 (carries the byte offset)."""

    def __init__(self, msg, offset=0):
        super().__init__(msg)
        self.offset = int(offset)


class SizeError(Error):
    """errors.h:32-35"""


class EmptyModelError(Error):
    """errors.h:39-51 (carries the largest observed gradient magnitude)."""

    def __init__(self, msg, max_magnitude=0.0):
        super().__init__(msg)
        self.max_magnitude = float(max_magnitude)


class BoundsError(Error):
    """errors.h:54-57"""


class BudgetError(Error):
    """errors.h:60-63"""


class GeometryError(Error):
    """errors.h:66-69"""


class InvalidArgument(Error, ValueError):
    """errors.h:72-75"""


class CudaError(Error):
    """Device missing or CUDA runtime failure (no reference counterpart)."""


class NcclError(Error):
    """NCCL missing or a collective failed (multi-GPU path; no reference counterpart)."""


_BY_STATUS = {
    abi.EA_ERR_INVALID_ARGUMENT: InvalidArgument,
    abi.EA_ERR_SIZE: SizeError,
    abi.EA_ERR_BOUNDS: BoundsError,
    abi.EA_ERR_BUDGET: BudgetError,
    abi.EA_ERR_GEOMETRY: GeometryError,
    abi.EA_ERR_CUDA: CudaError,
    abi.EA_ERR_NCCL: NcclError,
    abi.EA_ERR_INTERNAL: Error,
}


def raise_for_status(status, message, value=0.0):
    if status == abi.EA_OK:
        return
    if isinstance(message, bytes):
        message = message.decode("utf-8", "replace")
    if status == abi.EA_ERR_EMPTY_MODEL:
        raise EmptyModelError(message, value)
    if status == abi.EA_ERR_PARSE:
        raise ParseError(message, value)
    raise _BY_STATUS.get(status, Error)(message)

"""Exception types of the reference (include/sconv/errors.hpp:9-26, exec.hpp:43-51).

The C ABI returns integer statuses (include/sconv_cuda.h); ``raise_for`` maps
them back onto these classes so Python callers see the reference's error
behaviour: ShapeError for dimension mismatches, ConfigError for bad strides /
pool tilings, FormatError for corrupted ECR / PECR data.
"""


class ShapeError(RuntimeError):
    """Tensor/kernel/window dimension mismatch (errors.hpp:9-12)."""


class ConfigError(RuntimeError):
    """Invalid runtime configuration (errors.hpp:14-17)."""


class FormatError(RuntimeError):
    """Corrupted or inconsistent compressed data (errors.hpp:19-22)."""


class IoError(RuntimeError):
    """File I/O failure (errors.hpp:24-26)."""


class DispatchError(RuntimeError):
    """A work item failed; identifies (block, thread) (exec.hpp:43-51)."""

    def __init__(self, block: int, thread: int, what: str):
        super().__init__(f"work item failed at block {block}, thread {thread}: {what}")
        self.block = block
        self.thread = thread


class CudaError(RuntimeError):
    """Device / runtime failure inside libsconv_cuda."""


_BY_STATUS = {1: ShapeError, 2: ConfigError, 3: FormatError, 4: IoError, 6: CudaError,
              7: ValueError}


def raise_for(status: int, message: str) -> None:
    if status == 0:
        return
    if status == 5:
        raise DispatchError(-1, -1, message)
    raise _BY_STATUS.get(status, RuntimeError)(message)

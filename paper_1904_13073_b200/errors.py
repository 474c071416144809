"""dynsurf error hierarchy (reference: proj/core/include/dynsurf/errors.hpp:8-38).

The C ABI returns a ds_status; the host mirror rethrows the matching type.
"""


class Error(RuntimeError):
    """dynsurf::Error — also raised for numerical failures of the normal equations."""


class DimensionMismatch(Error):
    pass


class MissingInput(Error):
    pass


class CorruptFrame(Error):
    pass


class IoFailure(Error):
    pass


class EmptyGeometry(Error):
    pass


class UnknownScenario(Error):
    pass


class ConfigError(Error):
    pass


class CapacityExceeded(Error):
    """Device capacity (surfels / nodes / JtJ blocks) exceeded — B200 path only."""


class CudaError(Error):
    """CUDA runtime failure or no CUDA device (there is no CPU fallback)."""


class InvalidArgument(Error):
    pass


_BY_STATUS = {
    1: DimensionMismatch,
    2: EmptyGeometry,
    3: Error,
    4: ConfigError,
    5: CapacityExceeded,
    6: CudaError,
    7: InvalidArgument,
    8: UnknownScenario,
}


def from_status(status: int, msg: str) -> Error:
    return _BY_STATUS.get(int(status), Error)(msg or f"ds_status {status}")

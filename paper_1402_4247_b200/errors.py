"""Exception taxonomy mirroring kband (/root/reference/proj/include/kband/common.hpp:21-38).

C-ABI status codes (include/kbgrid.h) map one-to-one onto these classes.
"""


class Error(RuntimeError):
    status = -1


class ConfigError(Error):
    status = 1


class DimensionError(Error):
    status = 2


class ConsistencyError(Error):
    status = 3


class ConvergenceError(Error):
    """Non-finite values (kband raises ConvergenceError on NaN, householder.cpp:119-123)."""
    status = 4


class CudaError(Error):
    status = 5


class CollectiveError(Error):
    status = 6


_BY_STATUS = {c.status: c for c in (ConfigError, DimensionError, ConsistencyError, ConvergenceError,
                                    CudaError, CollectiveError)}


def raise_for_status(status: int, what: str, detail: str = "") -> None:
    if status == 0:
        return
    cls = _BY_STATUS.get(status, Error)
    msg = f"{what}: {detail}" if detail else f"{what} failed with status {status}"
    raise cls(msg)

"""Error taxonomy mirroring the reference (pkg/src/sinkloss/errors.py:6-83).

The C ABI returns integer statuses (ffi.ts:21-25 plus extensions); the
Python layer raises the reference's exception for each, so callers written
against ``sinkloss`` catch the same types.
"""

from __future__ import annotations

from . import _lib


class SinklossError(Exception):
    """Base class for all package errors (errors.py:6-7)."""

    status: int | None = None


class ShapeMismatch(SinklossError):
    """Batched array shapes disagree (errors.py:55-56); status 10."""

    status = _lib.STATUS_SHAPE_MISMATCH


class DimensionMismatch(SinklossError):
    """Histogram / cost dimensions disagree (errors.py:51-52)."""


class InvalidHistogram(SinklossError):
    """A histogram row is non-finite, negative or not normalised; status 11.

    The reference distinguishes NonFinite / NegativeMass / NotNormalised
    (errors.py:10-30); the device validator reports the first offending row.
    """

    status = _lib.STATUS_INVALID_HISTOGRAM

    def __init__(self, message: str, row: int | None = None):
        self.row = row
        super().__init__(message)


class NonFinite(InvalidHistogram):
    """errors.py:10-15."""


class NegativeMass(InvalidHistogram):
    """errors.py:18-23."""


class NotNormalised(InvalidHistogram):
    """errors.py:26-31."""


class NaNProduced(SinklossError):
    """Non-finite solver state or output (errors.py:38-39); status 12."""

    status = _lib.STATUS_NON_FINITE_OUTPUT


class ZeroMassGradient(SinklossError):
    """Gradient requested for a lane with a zero-mass bin (errors.py:59-68); status 13."""

    status = _lib.STATUS_ZERO_MASS_LANE

    def __init__(self, lane: int | None = None):
        self.lane = lane
        where = "" if lane is None else f" in lane {lane}"
        super().__init__(f"zero-mass bin{where}: gradient undefined")


class InvalidConfig(SinklossError, ValueError):
    """SinkhornConfig validation (core.py:88-96 raises ValueError); status 14."""

    status = _lib.STATUS_INVALID_CONFIG


class InvalidCost(SinklossError, ValueError):
    """CostMatrix validation (core.py:53-63 raises ValueError); status 15."""

    status = _lib.STATUS_INVALID_COST


class DeviceError(SinklossError, RuntimeError):
    """CUDA failure, bad argument or workspace error inside the library (16-20)."""


_BY_STATUS = {
    _lib.STATUS_SHAPE_MISMATCH: ShapeMismatch,
    _lib.STATUS_INVALID_HISTOGRAM: InvalidHistogram,
    _lib.STATUS_NON_FINITE_OUTPUT: NaNProduced,
    _lib.STATUS_INVALID_CONFIG: InvalidConfig,
    _lib.STATUS_INVALID_COST: InvalidCost,
}


def raise_for_status(status: int, what: str, lane: int | None = None) -> None:
    """Translate a C-ABI status into the reference's exception (loss.ts:93-95)."""
    if status == _lib.STATUS_OK:
        return
    detail = _lib.last_error()
    if status == _lib.STATUS_ZERO_MASS_LANE:
        raise ZeroMassGradient(lane)
    cls = _BY_STATUS.get(status, DeviceError)
    raise cls(f"{what} failed with status {status}: {detail}")

"""Exception vocabulary of the reference (include/dagsplit/errors.hpp:8-43,
graph.hpp:239-241), mapped from the C-ABI status codes (dsg_b200.h)."""
from __future__ import annotations

from . import _abi


class DagsplitError(RuntimeError):
    pass


class InfeasibleError(DagsplitError):
    """errors.hpp:8-10."""

    def __init__(self, msg: str = "no feasible assignment exists"):
        super().__init__(msg)


class DeadlineExceeded(DagsplitError):
    """errors.hpp:12-14."""

    def __init__(self, msg: str = "time limit reached"):
        super().__init__(msg)


class MissingBandwidth(DagsplitError):
    """errors.hpp:21-24."""

    def __init__(self, msg: str = "replication requires a bandwidth value"):
        super().__init__(msg)


class IdealBudgetExceeded(Exception):
    """graph.hpp:239-241 (deliberately not a DagsplitError, like the reference
    struct that is not a std::exception)."""

    def __init__(self, limit: int):
        super().__init__(f"ideal budget {limit} exceeded")
        self.limit = limit


class DeviceError(DagsplitError):
    """No reference analogue: the CUDA library or device failed."""


class Unsupported(DagsplitError):
    """A valid request this build does not implement on the device."""


def raise_for_status(status: int, message: bytes, budget_limit: int = 0) -> None:
    msg = message.decode(errors="replace") if isinstance(message, (bytes, bytearray)) else str(message)
    if status == _abi.DSG_OK:
        return
    if status == _abi.DSG_INFEASIBLE:
        raise InfeasibleError()
    if status == _abi.DSG_DEADLINE:
        raise DeadlineExceeded()
    if status == _abi.DSG_BUDGET:
        raise IdealBudgetExceeded(budget_limit)
    if status == _abi.DSG_MISSING_BANDWIDTH:
        raise MissingBandwidth()
    if status == _abi.DSG_INVALID:
        raise ValueError(msg)  # std::invalid_argument / std::domain_error
    if status == _abi.DSG_OVERFLOW:
        raise OverflowError(msg)  # std::overflow_error
    if status == _abi.DSG_LOGIC:
        raise RuntimeError(msg)  # std::logic_error
    if status == _abi.DSG_UNSUPPORTED:
        raise Unsupported(msg)
    raise DeviceError(msg or f"status {status}")

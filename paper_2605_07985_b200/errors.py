"""Error types raised at the hot-path boundary.

Names, constructor signatures and meaning follow the reference hierarchy
(`pkg/src/dooly/errors.py:4-85`); the taint / trace / opset classes serve the
record producer (tracer.py, opset.py) that feeds dedup.  C-ABI status
codes (include/dooly_b200.h) map onto these one-to-one in ``raise_for_status``.
"""

from __future__ import annotations


class DoolyError(Exception):
    """Root of every error this package raises (errors.py:4)."""


class MixValueConflict(DoolyError):
    """One value would carry two labels inside a Mix taint (errors.py:8)."""


class UnknownComponent(DoolyError):
    """split() of a Mix by a value it does not contain (errors.py:12)."""


class ShapeMismatch(DoolyError):
    """A reshape whose element counts disagree (errors.py:28)."""


class MalformedTrace(DoolyError):
    """Trace events whose intervals do not nest (errors.py:32)."""


class RetraceFailed(DoolyError):
    """Two consecutive dummy batches both collided with model values (errors.py:36)."""


class ContextUnavailable(DoolyError):
    """Context emulation asked for a stateless entry (errors.py:40)."""


class Unresolvable(DoolyError):
    """No runnable ancestor covers a kernel, not even the root (errors.py:44)."""


class ParseError(DoolyError):
    """Manifest / workload / trace file is not the documented format (errors.py:16)."""


class ValidationError(DoolyError):
    """Parsed document violates an invariant; ``path`` names the field (errors.py:20-25)."""

    def __init__(self, path: str, message: str):
        super().__init__(f"{path}: {message}")
        self.path = path


class StoreUnavailable(DoolyError):
    """The latency database could not be reached (errors.py:48)."""


class DuplicateKey(DoolyError):
    """Measurement key re-inserted with a different latency (errors.py:52)."""


class OraclePanic(DoolyError):
    """The analytical latency model failed at a sweep point (errors.py:56)."""


class InsufficientData(DoolyError):
    """Too few measurements to fit a signature (errors.py:60-69)."""

    def __init__(self, signature_hash: str, have: int, need: int):
        super().__init__(
            f"signature {signature_hash[:12]}…: {have} measurements, need >= {need}"
        )
        self.signature_hash = signature_hash
        self.have = have
        self.need = need


class UnknownSignature(DoolyError):
    """Prediction requested for an unfitted signature (errors.py:72)."""


class LengthMismatch(DoolyError):
    """Series of unequal length compared (errors.py:76)."""


class ZeroTruth(DoolyError):
    """MAPE requested against a series containing zero (errors.py:80)."""


class NonTermination(DoolyError):
    """Simulation exceeded its iteration cap (errors.py:84)."""


class DeviceError(DoolyError):
    """A CUDA call inside libdooly_b200 failed (status DOOLY_ERR_CUDA)."""


class CommError(DoolyError):
    """An NCCL call inside libdooly_b200 failed (status DOOLY_ERR_NCCL)."""


# C-ABI status codes (include/dooly_b200.h) -> exception class.
STATUS_OK = 0
STATUS_INVALID_ARG = 1
STATUS_INSUFFICIENT_DATA = 2
STATUS_UNKNOWN_SIGNATURE = 3
STATUS_DUPLICATE_KEY = 4
STATUS_NON_TERMINATION = 5
STATUS_CUDA = 6
STATUS_NCCL = 7

_STATUS_CLASS = {
    STATUS_INVALID_ARG: ValueError,
    STATUS_UNKNOWN_SIGNATURE: UnknownSignature,
    STATUS_DUPLICATE_KEY: DuplicateKey,
    STATUS_NON_TERMINATION: NonTermination,
    STATUS_CUDA: DeviceError,
    STATUS_NCCL: CommError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == STATUS_OK:
        return
    cls = _STATUS_CLASS.get(code, DoolyError)
    raise cls(message)

"""Exception classes of the drop-in API.

Same class names and meanings as the reference's taxonomy
(pkg/src/deflamg/errors.py:4-37), so callers catching ``deflamg`` errors by
name keep working.  The C ABI returns negative status codes
(include/dflb200.h, ``DFL_E_*``); :func:`raise_for_status` maps them here.
"""


class DeflamgError(Exception):
    """Root of every error this package raises."""


class DimensionError(DeflamgError):
    """Operand shapes do not fit together."""


class StructureError(DeflamgError):
    """A matrix breaks a structural precondition (zero diagonal, bad CSR)."""


class SingularMatrixError(DeflamgError):
    """A dense factorisation met a (numerically) zero pivot."""


class PartitionError(DeflamgError):
    """A row partition is malformed or does not match the matrix."""


class CommunicatorError(DeflamgError):
    """A collective / halo exchange failed or was called inconsistently."""


class BreakdownError(DeflamgError):
    """Krylov breakdown (kept for API parity; solvers report, not raise)."""


class ParseError(DeflamgError):
    """Input file could not be parsed."""


class ConfigError(DeflamgError):
    """Unknown configuration key or badly typed value."""


class DeviceError(DeflamgError):
    """CUDA / NCCL failure, or the native library is missing on this host."""


# status codes shared with include/dflb200.h
_STATUS = {
    -1: DimensionError,
    -2: StructureError,
    -3: SingularMatrixError,
    -4: PartitionError,
    -5: CommunicatorError,
    -6: ConfigError,
    -7: DeviceError,
    -8: DeviceError,
    -9: ParseError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == 0:
        return
    cls = _STATUS.get(code, DeflamgError)
    raise cls(message or f"native call failed with status {code}")

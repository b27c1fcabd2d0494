"""Error taxonomy of the drop-in boundary.

The class names are those of the reference package (F/errors.py:4-57) so
callers' `except` clauses keep working; each C-ABI status code of
include/ls2.h maps onto one of them (see STATUS_TO_ERROR).
"""

from __future__ import annotations


class FtrainError(Exception):
    """Root of every error raised by this package."""


class ShapeMismatch(FtrainError):
    """Operand shapes, dtypes or ranks that the operator cannot accept."""


class TokenOutOfRange(FtrainError):
    """A token id outside [0, vocab)."""


class SequenceTooLong(FtrainError):
    """A batch longer than the positional table."""


class DegenerateRow(FtrainError):
    """LayerNorm row with zero variance while eps == 0."""


class AllMaskedRow(FtrainError):
    """Softmax row in which every position is masked."""


class TargetOutOfRange(FtrainError):
    """Criterion target outside [0, V)."""


class IncompleteGradientSet(FtrainError):
    """Packed cross-attention backward requested before all decoder layers ran."""


class DuplicateName(FtrainError):
    """Workspace parameter name registered twice."""


class NonFiniteGradient(FtrainError):
    """Raised only where skipping the step is impossible."""


class UntaggedTensor(FtrainError):
    """Memory-plan tensor without a known kind."""


class ParseError(FtrainError):
    """Malformed input file."""


class ConfigError(FtrainError):
    """Invalid configuration value."""


class DataError(FtrainError):
    """Unusable data source."""


class DeviceError(FtrainError):
    """CUDA / cuBLAS runtime failure inside the native library (no CPU fallback)."""


# include/ls2.h status codes -> exception classes
STATUS_TO_ERROR = {
    1: ShapeMismatch,
    2: TokenOutOfRange,
    3: SequenceTooLong,
    4: DegenerateRow,
    5: AllMaskedRow,
    6: TargetOutOfRange,
    7: ShapeMismatch,
    8: DeviceError,
    9: DeviceError,
}

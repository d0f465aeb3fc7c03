"""Error types of the inference path, mirroring pkg/src/cuppl/errors.py.

Same class names, `kind` strings and render() format (errors.py:6-20) so code written
against the reference catches the same exceptions. Only the runtime/inference part of the
hierarchy exists here; compile-time errors belong to the (out-of-scope) frontend.
"""

from __future__ import annotations


class CupError(Exception):
    """Base class (cuppl/errors.py:6-20)."""

    kind = "error"

    def __init__(self, message, span=None):
        super().__init__(message)
        self.message = message
        self.span = span

    def render(self):
        if self.span is not None:
            s = self.span
            return f"error: {self.kind} at {s.file}:{s.start_line}:{s.start_col}: {self.message}"
        return f"error: {self.kind}: {self.message}"


class CupRuntimeError(CupError):  # errors.py:73
    kind = "runtime-error"


class TypeMismatchError(CupRuntimeError):  # errors.py:93
    kind = "value-type-mismatch"


class UnsupportedDistError(CupRuntimeError):  # errors.py:97
    kind = "unsupported-distribution"


class InvalidDistParamError(CupRuntimeError):  # errors.py:135
    kind = "invalid-dist-parameter"


class InferError(CupError):  # errors.py:111
    kind = "inference-error"


class ContinuousDistError(InferError):  # errors.py:115
    kind = "continuous-distribution"


class AllZeroWeightError(InferError):  # errors.py:119
    kind = "all-zero-weights"


class InferRuntimeError(InferError):  # errors.py:123-132
    """Wraps a runtime failure inside an engine run with its provenance."""

    kind = "inference-runtime-error"

    def __init__(self, message, cause=None, seed=None, step=None):
        super().__init__(message)
        self.cause = cause
        self.seed = seed
        self.step = step


class NativeLibraryError(CupRuntimeError):
    """libcuppl_gpu.so is missing or a CUDA call failed. There is no CPU fallback."""

    kind = "native-library"

"""Exception types (mirror of moetrim/errors.py:1-9)."""


class ValidationError(ValueError):
    """An input violates a documented precondition (moetrim.errors.ValidationError)."""


class TraceFormatError(ValidationError):
    """A persisted trace file is malformed (moetrim.errors.TraceFormatError)."""


class NativeLibraryError(RuntimeError):
    """liblynx_b200.so is missing, failed to load, or a CUDA call failed.

    Raised instead of silently falling back to a CPU path: this package has
    no CPU implementation of the hot path.
    """

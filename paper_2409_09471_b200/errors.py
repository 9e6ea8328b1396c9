"""Exception types mirroring the reference (tt.py:22-27, streaming.py:20-21)."""


class ShapeMismatch(ValueError):
    """Operands have incompatible mode sizes or rank chains (tt.py:22-23)."""


class SizeLimit(ValueError):
    """A dense materialization would exceed the configured entry cap (tt.py:26-27)."""


class DegenerateRecovery(ValueError):
    """Recovery hit an all-zero cross matrix against nonzero sketches (streaming.py:20-21)."""

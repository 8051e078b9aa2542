"""Error taxonomy of the reference (TEST INFRASTRUCTURE ONLY).

Restates ``chainscan/core.py:30-44`` (StructuralError, ChainDivergedError) and
``chainscan/noise.py:30-31`` (ConfigurationError).
"""


class ConfigurationError(ValueError):
    """Bad configuration / undeclared noise slot (noise.py:30)."""


class StructuralError(ValueError):
    """Shape or variant mismatch (core.py:30)."""


class ChainDivergedError(RuntimeError):
    """Non-finite state or divergence guard (core.py:34-44)."""

    def __init__(self, message, step=None, iteration=None):
        super().__init__(message)
        self.step = step
        self.iteration = iteration

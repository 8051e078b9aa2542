"""Exception types of the reference API (chainscan/core.py:30-44, noise.py:30)."""


class ConfigurationError(ValueError):
    """A slot/layout/config request the solver was not declared with."""


class StructuralError(ValueError):
    """Shape or variant mismatch between values that must agree."""


class ChainDivergedError(RuntimeError):
    """A solver or sampler produced a non-finite state (carries step, iteration)."""

    def __init__(self, message, step=None, iteration=None):
        super().__init__(message)
        self.step = step
        self.iteration = iteration

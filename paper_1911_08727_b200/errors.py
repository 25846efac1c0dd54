"""Exception types of the drop-in surface (same names and bases as R: errors.py:4-13)."""


class StructureError(ValueError):
    """Layer layouts disagree or a structural input is malformed."""


class DivergenceError(ArithmeticError):
    """Training produced a non-finite quantity."""

    def __init__(self, message: str, iteration: int | None = None):
        super().__init__(message)
        self.iteration = iteration

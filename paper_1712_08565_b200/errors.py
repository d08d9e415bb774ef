"""Exception types mirroring the reference (same names and meaning)."""


class WQConstructionError(RuntimeError):
    """wq.py:29-39: an exactness system of some row cannot be satisfied."""

    def __init__(self, row, residual, msg=None):
        self.row = row
        self.residual = residual
        super().__init__(msg or f"exactness system for row {row} unsolvable (residual {residual:.3e})")


class DegenerateGeometryError(RuntimeError):
    """operators.py:25-31: non-positive Jacobian determinant."""

    def __init__(self, point, det, msg=None):
        self.point = point
        self.det = det
        super().__init__(msg or f"non-positive Jacobian determinant {det:.3e} at parametric point {point}")


class IndefiniteOperatorError(RuntimeError):
    """solvers.py:24."""


class EigenSolveError(RuntimeError):
    """solvers.py:28."""

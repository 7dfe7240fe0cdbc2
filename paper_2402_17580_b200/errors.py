"""Convergence errors of the implicit scheme (batch.py:74-79,
integrator.py:119-128)."""

__all__ = ["BatchConvergenceError", "FixedPointDivergence"]


class BatchConvergenceError(RuntimeError):
    """Implicit fixed-point iteration failed (batch.py:74-79)."""

    def __init__(self, indices, message=None):
        self.indices = list(indices)
        super().__init__(message or
                         f"fixed-point iteration failed at point indices {self.indices}")


class FixedPointDivergence(BatchConvergenceError):
    """Crank-Nicolson fixed-point iteration failed; carries the last iterate
    and its WRMS residual norm (integrator.py:119-128)."""

    def __init__(self, state, residual_norm, iters):
        self.state = state
        self.residual_norm = residual_norm
        self.iters = iters
        super().__init__([0], f"no convergence after {iters} iterations "
                              f"(WRMS residual {residual_norm:.3e}); last iterate {state}")

"""Solver settings — mirror of the reference's ``SolveSettings``
(/root/reference/pkg/src/fusedmpc/ilqr.py:27-60): same fields, defaults and
validation errors."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

DEFAULT_ALPHAS = (1.0, 0.5, 0.25, 0.1)  # ilqr.py:27


@dataclass(frozen=True)
class SolveSettings:
    """Horizon, bounds and iteration limits for a solve."""

    T: int
    u_min: np.ndarray
    u_max: np.ndarray
    K_max: int = 10
    alphas: tuple = DEFAULT_ALPHAS
    conv_tol: float = 1e-6
    boxqp_max_iter: int = 20
    boxqp_tol: float = 1e-9

    def __post_init__(self):
        object.__setattr__(self, "u_min", np.atleast_1d(np.asarray(self.u_min, dtype=np.float64)))
        object.__setattr__(self, "u_max", np.atleast_1d(np.asarray(self.u_max, dtype=np.float64)))
        if self.T < 1:
            raise ConfigError(f"horizon T must be >= 1, got {self.T}")
        if self.K_max < 1:
            raise ConfigError(f"K_max must be >= 1, got {self.K_max}")
        if not np.all(self.u_min < self.u_max):
            raise ConfigError("u_min must be elementwise below u_max")
        a = np.asarray(self.alphas, dtype=np.float64)
        if a.size == 0 or np.any(a <= 0.0) or np.any(a > 1.0) or np.any(np.diff(a) >= 0.0):
            raise ConfigError("alphas must be a strictly decreasing sequence in (0, 1]")
        object.__setattr__(self, "alphas", tuple(float(v) for v in a))

    def bounds_for(self, n_u: int):
        """Bounds broadcast to the control dimension (ilqr.py:56-60)."""
        try:
            lo = np.broadcast_to(self.u_min, (n_u,)).astype(np.float64)
            hi = np.broadcast_to(self.u_max, (n_u,)).astype(np.float64)
        except ValueError as e:
            raise ConfigError(f"bounds do not broadcast to n_u={n_u}") from e
        return np.ascontiguousarray(lo), np.ascontiguousarray(hi)

    def replace(self, **kw) -> "SolveSettings":
        d = dict(T=self.T, u_min=self.u_min, u_max=self.u_max, K_max=self.K_max, alphas=self.alphas,
                 conv_tol=self.conv_tol, boxqp_max_iter=self.boxqp_max_iter, boxqp_tol=self.boxqp_tol)
        d.update(kw)
        return SolveSettings(**d)

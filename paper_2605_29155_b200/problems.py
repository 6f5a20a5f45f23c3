"""Synthetic problem generators (host-side numpy), shared by tests, goldens and bench.

``hover_problem`` follows the reference's ``make_hover_problem``
(/root/reference/pkg/src/fusedmpc/batchexec.py:215-233) for the planar quadrotor
and its 13-state analogue from SURVEY.md §8(d); ``random_problem`` follows the
reference's random-cost batches (tests/test_acceptance.py:139-155,
tests/test_batchexec.py:20-32), which leave ~25% of control entries on a bound.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dynamics import KIND_PLANAR_QUADROTOR, KIND_QUADROTOR13, DynModel
from .settings import SolveSettings


@dataclass
class Problem:
    model: DynModel
    settings: SolveSettings
    x0: np.ndarray      # (B, nx)
    diag: np.ndarray    # (B, T, nz) diagonal of C_t
    c: np.ndarray       # (B, T, nz)
    U_warm: np.ndarray  # (B, T, nu)

    @property
    def B(self):
        return self.x0.shape[0]

    def slice(self, lo: int, hi: int) -> "Problem":
        """Problems [lo, hi) of the batch (a rank's shard of a global batch)."""
        return Problem(self.model, self.settings, self.x0[lo:hi], self.diag[lo:hi], self.c[lo:hi],
                       self.U_warm[lo:hi])

    def dense_C(self) -> np.ndarray:
        """(B, T, nz, nz) with the diagonal placed as StageCostParams.from_diag does."""
        B, T, nz = self.diag.shape
        C = np.zeros((B, T, nz, nz))
        idx = np.arange(nz)
        C[:, :, idx, idx] = self.diag
        return C


def default_model(kind: int) -> DynModel:
    if kind == KIND_QUADROTOR13:
        return DynModel.quadrotor(dt=0.05)
    return DynModel.planar_quadrotor(dt=0.05)


def hover_bounds(model: DynModel):
    n_u = model.n_u
    if model.kind == KIND_PLANAR_QUADROTOR:
        return np.zeros(n_u), np.full(n_u, 2.0 * model.mass * model.gravity)
    return np.zeros(n_u), np.full(n_u, model.mass * model.gravity)


def hover_problem(model: DynModel, B: int, T: int, seed: int = 0, **settings_kw) -> Problem:
    rng = np.random.default_rng(seed)
    n_x, n_u = model.n_x, model.n_u
    n_z = n_x + n_u
    u_h = model.hover_control()
    lo, hi = hover_bounds(model)
    kw = dict(T=T, u_min=lo, u_max=hi)
    kw.update(settings_kw)
    settings = SolveSettings(**kw)
    if model.kind == KIND_PLANAR_QUADROTOR:
        d = np.array([1.0, 1.0, 1.0, 0.1, 0.1, 0.1, 0.05, 0.05])
        c1 = np.zeros(n_z)
        c1[n_x:] = -d[n_x:] * u_h
        x0 = np.zeros((B, n_x))
        x0[:, 0:2] = rng.uniform(-1.0, 1.0, size=(B, 2))
        x0[:, 3:5] = rng.uniform(-0.5, 0.5, size=(B, 2))
    elif model.kind == KIND_QUADROTOR13:
        d = np.concatenate([np.full(3, 1.0), np.full(4, 1.0), np.full(3, 0.1), np.full(3, 0.1),
                            np.full(4, 0.05)])
        z_ref = np.concatenate([np.zeros(3), [1.0, 0.0, 0.0, 0.0], np.zeros(6), u_h])
        c1 = -d * z_ref
        x0 = np.zeros((B, n_x))
        x0[:, 0:3] = rng.uniform(-1.0, 1.0, size=(B, 3))
        x0[:, 3] = 1.0
        x0[:, 7:10] = rng.uniform(-0.5, 0.5, size=(B, 3))
    else:
        raise ValueError("hover_problem supports the planar and 13-state quadrotors")
    diag = np.broadcast_to(d, (B, T, n_z)).copy()
    c = np.broadcast_to(c1, (B, T, n_z)).copy()
    U_warm = np.broadcast_to(u_h, (B, T, n_u)).copy()
    return Problem(model, settings, x0, diag, c, U_warm)


def random_problem(model: DynModel, B: int, T: int, seed: int = 104, **settings_kw) -> Problem:
    rng = np.random.default_rng(seed)
    n_x, n_u = model.n_x, model.n_u
    n_z = n_x + n_u
    if model.kind == KIND_PLANAR_QUADROTOR:
        lo, hi = np.zeros(n_u), np.full(n_u, 12.0)
    else:
        lo, hi = hover_bounds(model)
    kw = dict(T=T, u_min=lo, u_max=hi)
    kw.update(settings_kw)
    settings = SolveSettings(**kw)
    diag = rng.uniform(0.05, 2.0, size=(B, T, n_z))
    c = rng.normal(size=(B, T, n_z))
    x0 = 0.5 * rng.normal(size=(B, n_x))
    if model.kind == KIND_QUADROTOR13:
        q = np.array([1.0, 0.0, 0.0, 0.0]) + 0.1 * rng.normal(size=(B, 4))
        x0[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    U_warm = rng.uniform(0.0, 1.0, size=(B, T, n_u)) * hi
    return Problem(model, settings, x0, diag, c, U_warm)

"""Object-level API mirroring the reference's single-instance and batch wrappers, on the
B200 kernels:

    ilqr.solve / SolveResult / Gains                      (ilqr.py:63-82, 414-440)
    gradlayer.backward / BackwardSeed / GradOutput       (gradlayer.py:30-50, 166-182)
    batchexec.BatchProblem / solve_batch / backward_batch / make_hover_problem
                                                          (batchexec.py:42-63, 166-233)

Semantics follow the reference: float64 by default; the single-instance ``solve`` raises
DivergenceError when the initial rollout diverges (or every line-search candidate does) and
NumericError when a stage Hessian is not positive definite; ``backward`` raises NumericError
on a singular reduced stage Hessian and flags a non-converged forward solve as
``approximate``; the batch calls never raise per instance, they flag ``failed``.
``lin`` arguments are accepted for signature compatibility — the backward kernel
relinearises at the solution itself (policy.py:257-272). Each call is one kernel launch
(two for solve + backward) regardless of B.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import problems as _problems
from . import solver as _solver
from .dynamics import DynModel
from .errors import ConfigError, DivergenceError, NumericError
from .qcost import StageCostParams, Trajectory, stack
from .settings import SolveSettings


@dataclass(frozen=True)
class Gains:
    K: np.ndarray  # (T, n_u, n_x)
    k: np.ndarray  # (T, n_u)


@dataclass(frozen=True)
class SolveResult:
    traj: Trajectory
    gains: Gains
    cost: float
    iterations: int
    converged: bool
    clamped_mask: np.ndarray  # (T, n_u) bool
    alpha_history: np.ndarray  # accepted step per executed iteration (0 = no step)
    failed: bool = False
    fail_stage: int = -1
    model: DynModel = field(default=None, repr=False, compare=False)
    settings: SolveSettings = field(default=None, repr=False, compare=False)


@dataclass(frozen=True)
class BackwardSeed:
    dL_dX: np.ndarray  # (T+1, n_x)
    dL_dU: np.ndarray  # (T, n_u)

    def __post_init__(self):
        object.__setattr__(self, "dL_dX", np.ascontiguousarray(self.dL_dX, dtype=np.float64))
        object.__setattr__(self, "dL_dU", np.ascontiguousarray(self.dL_dU, dtype=np.float64))
        if self.dL_dX.shape[0] != self.dL_dU.shape[0] + 1:
            raise ConfigError("seed must have T+1 state rows and T control rows")


@dataclass(frozen=True)
class GradOutput:
    dC: np.ndarray  # (T, n_z, n_z)
    dc: np.ndarray  # (T, n_z)
    dx_init: np.ndarray  # (n_x,)
    approximate: bool = False
    failed: bool = False


@dataclass(frozen=True)
class BatchProblem:
    """B instances sharing model, horizon and bounds (batchexec.py:42-63)."""

    model: DynModel
    x_init: np.ndarray  # (B, n_x)
    params: list  # B StageCostParams
    U_warm: np.ndarray  # (B, T, n_u)
    settings: SolveSettings

    def __post_init__(self):
        B = self.x_init.shape[0]
        if B < 1:
            raise ConfigError("batch must contain at least one instance")
        if len(self.params) != B or self.U_warm.shape[0] != B:
            raise ConfigError("x_init, params and U_warm must agree on batch size")

    @property
    def B(self) -> int:
        return self.x_init.shape[0]


def _collect(model, settings, out) -> list:
    """Per-instance SolveResults from a device SolveOutput (ilqr.collect_result, ilqr.py:250-268)."""
    X, U, J = _solver.to_numpy(out.X), _solver.to_numpy(out.U), _solver.to_numpy(out.J)
    K, k = _solver.to_numpy(out.K), _solver.to_numpy(out.k)
    it, conv = _solver.to_numpy(out.iters), _solver.to_numpy(out.converged)
    div, ft = _solver.to_numpy(out.diverged), _solver.to_numpy(out.fail_t)
    ah = _solver.to_numpy(out.alpha_hist)
    lo, hi = settings.bounds_for(model.n_u)
    res = []
    for i in range(X.shape[0]):
        failed = bool(ft[i] >= 0) or bool(div[i])
        n_it = int(it[i])
        res.append(SolveResult(
            traj=Trajectory(X[i].astype(np.float64), U[i].astype(np.float64)),
            gains=Gains(K[i].astype(np.float64), k[i].astype(np.float64)), cost=float(J[i]), iterations=n_it,
            converged=bool(conv[i]) and not failed, clamped_mask=(U[i] <= lo) | (U[i] >= hi),
            alpha_history=ah[i, :n_it].astype(np.float64), failed=failed, fail_stage=int(ft[i]),
            model=model, settings=settings))
    return res, it, div, ft


def solve(model: DynModel, x_init, p: StageCostParams, U_warm, settings: SolveSettings,
          dtype=torch.float64, device=None) -> SolveResult:
    """Single-instance solve (ilqr.solve, ilqr.py:414-440)."""
    x_init = np.ascontiguousarray(x_init, dtype=np.float64)
    U_warm = np.ascontiguousarray(U_warm, dtype=np.float64)
    if p.T != settings.T:
        raise ConfigError(f"cost horizon {p.T} != settings horizon {settings.T}")
    if U_warm.shape != (settings.T, model.n_u):
        raise ConfigError(f"U_warm must be ({settings.T}, {model.n_u}), got {U_warm.shape}")
    if p.n_x != model.n_x:
        raise ConfigError(f"cost n_x={p.n_x} does not match model n_x={model.n_x}")
    out = _solver.solve_raw(model, settings, x_init[None], p.C[None], p.c[None], U_warm[None], dtype=dtype,
                            device=device)
    res, it, div, ft = _collect(model, settings, out)
    if ft[0] >= 0 and div[0] and it[0] == 0:
        raise DivergenceError("initial rollout diverged", stage=int(ft[0]))
    if ft[0] >= 0 and not div[0]:
        raise NumericError("stage Hessian not positive definite", stage=int(ft[0]))
    if div[0] and it[0] > 0:
        raise DivergenceError("all line-search candidates diverged")
    return res[0]


def _grads(results, params, seeds, dtype, device):
    model, settings = results[0].model, results[0].settings
    if model is None or settings is None:
        raise ConfigError("results must come from api.solve / api.solve_batch")
    C, c = stack(params)
    X = np.stack([r.traj.X for r in results])
    U = np.stack([r.traj.U for r in results])
    dX = np.stack([s.dL_dX for s in seeds])
    dU = np.stack([s.dL_dU for s in seeds])
    g = _solver.backward_raw(model, settings, C, c, X, U, dX, dU, dtype=dtype, device=device)
    return _solver.to_numpy(g.dC), _solver.to_numpy(g.dc), _solver.to_numpy(g.dx0), _solver.to_numpy(g.fail_t)


def backward(result: SolveResult, lin, p: StageCostParams, seed: BackwardSeed, dtype=torch.float64,
             device=None) -> GradOutput:
    """Differentiate a loss through one solve (gradlayer.backward, gradlayer.py:166-182)."""
    dC, dc, dx0, ft = _grads([result], [p], [seed], dtype, device)
    if ft[0] >= 0:
        raise NumericError("singular reduced stage Hessian", stage=int(ft[0]))
    return GradOutput(dC=dC[0], dc=dc[0], dx_init=dx0[0], approximate=not result.converged)


def solve_batch(prob: BatchProblem, mode="fused", pool=None, dtype=torch.float64, device=None):
    """Solve B instances (batchexec.solve_batch, batchexec.py:166-177); failures are flagged,
    not raised. Returns (list of SolveResult, stats)."""
    if mode not in ("fused", "naive"):
        raise ConfigError(f"mode must be one of ('fused', 'naive'), got {mode!r}")
    C, c = stack(prob.params)
    out = _solver.solve_raw(prob.model, prob.settings, prob.x_init, C, c, prob.U_warm, dtype=dtype, device=device)
    res, it, _, _ = _collect(prob.model, prob.settings, out)
    return res, {"total_dispatches": 1, "iterations": it}


def backward_batch(results, lins, params, seeds, mode="fused", pool=None, dtype=torch.float64, device=None):
    """Per-instance implicit differentiation over a solved batch (batchexec.backward_batch,
    batchexec.py:189-211); singular instances come back ``failed`` with zero gradients."""
    B = len(results)
    if not (len(params) == len(seeds) == B) or (lins is not None and len(lins) != B):
        raise ConfigError("results, lins, params and seeds must have equal length")
    dC, dc, dx0, ft = _grads(results, params, seeds, dtype, device)
    return [GradOutput(dC=dC[i], dc=dc[i], dx_init=dx0[i], approximate=not results[i].converged,
                       failed=bool(ft[i] >= 0)) for i in range(B)]


def make_hover_problem(B: int, T: int, settings_kw=None, seed: int = 0) -> BatchProblem:
    """Planar-quadrotor hover batch (batchexec.make_hover_problem, batchexec.py:215-233)."""
    model = DynModel.planar_quadrotor(dt=0.05)
    pb = _problems.hover_problem(model, B, T, seed=seed, **(settings_kw or {}))
    params = [StageCostParams.from_diag(pb.diag[i], pb.c[i], model.n_x) for i in range(B)]
    return BatchProblem(model, pb.x0, params, pb.U_warm, pb.settings)

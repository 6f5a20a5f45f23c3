"""AC-MPC drop-in: ``MpcSolver`` / ``MpcSolveLayer`` / ``mpc_control`` with the reference's
signatures and semantics (/root/reference/pkg/src/fusedmpc/policy.py:179-290), running on
the B200 kernels.

Differences a caller can observe, all deliberate:
  * the solve runs in the solver's dtype on the GPU (MpcSolver(dtype=torch.float32) by
    default; torch.float64 reproduces the reference's float64 solve, policy.py:235-236);
  * solver state (warm starts, the workspace) stays device-resident as torch tensors;
  * ``pool`` / ``mode`` are accepted for signature compatibility: there is one fused
    kernel per forward solve and one per backward, whatever the mode.
"""

from __future__ import annotations

import numpy as np
import torch

from . import solver as _solver
from .errors import ConfigError


class MpcSolver:
    """Solver handle: model, horizon settings, device and warm starts (policy.py:179-222).

    Warm-start slots implement the receding-horizon shift: after each solve the stored
    control sequence advances one step, repeating the last entry (policy.py:206-212).
    """

    def __init__(self, model, settings, pool=None, mode="fused", n_slots=1, device=None,
                 dtype=torch.float32, kernel="throughput"):
        if mode not in ("fused", "naive"):
            raise ConfigError(f"mode must be one of ('fused', 'naive'), got {mode!r}")
        self.model = model
        self.settings = settings
        self.pool = pool
        self.mode = mode
        self.n_slots = n_slots
        self.device = _solver._device(device)
        self.dtype = dtype
        # One forward mapping for every batch size, so a minibatch re-solve reproduces the
        # rollout's controls bit for bit (importance ratio exactly 1, trainer.py:9-12).
        self.kernel = kernel
        u_min, u_max = settings.bounds_for(model.n_u)
        self.default_u = np.clip(model.hover_control(), u_min, u_max)
        self.warm = None
        self.reset_warm()

    def reset_warm(self, slots=None):
        du = torch.as_tensor(self.default_u, dtype=self.dtype, device=self.device)
        if self.warm is None:
            self.warm = du.expand(self.n_slots, self.settings.T, self.model.n_u).clone()
        elif slots is None:
            self.warm[:] = du
        else:
            self.warm[slots] = du

    def push_warm(self, U, slots=None):
        """Store the time-shifted solution for the next receding-horizon call."""
        U = torch.as_tensor(U, dtype=self.dtype, device=self.device)
        shifted = torch.cat([U[:, 1:], U[:, -1:]], dim=1)
        if slots is None:
            self.warm[:] = shifted
        else:
            self.warm[slots] = shifted

    def solve_diag(self, x_init, diag, cvec, U_warm, dtype=None):
        """Batched solve from the diagonal cost parameterisation (policy.py:214-222).

        Returns (ws, iterations, converged, alpha_history, stats) like the reference;
        ``ws`` is a device-resident SolveOutput (ws.X, ws.U, ws.J, ws.K, ws.k, ...).
        """
        dtype = dtype or self.dtype
        ws = _solver.solve_raw(self.model, self.settings, x_init, diag, cvec, U_warm, dtype=dtype,
                               device=self.device, kernel=self.kernel)
        stats = {"dispatches_per_iteration": None, "total_dispatches": 1}
        return ws, ws.iters, ws.converged, ws.alpha_hist, stats

    def solve_dense(self, x_init, C, c, U_warm, dtype=None):
        """Dense-cost counterpart (batchexec.solve_raw, batchexec.py:156-163)."""
        dtype = dtype or self.dtype
        ws = _solver.solve_raw(self.model, self.settings, x_init, C, c, U_warm, dtype=dtype, device=self.device,
                               kernel=self.kernel)
        return ws, ws.iters, ws.converged, ws.alpha_hist, {"total_dispatches": 1}


class MpcSolveLayer(torch.autograd.Function):
    """First optimal control of the batched solve as a differentiable op (policy.py:225-283).

    forward(diag (B,T,nz), cvec (B,T,nz), solver, x_init (B,n), U_warm (B,T,m), stats_sink)
        -> u0 (B,m) in diag.dtype on diag.device
    backward(grad_u0) -> (grad_diag, grad_c, None, None, None, None); the implicit sweep is
        seeded with dL/du_0 only and failed instances get zero gradients (policy.py:277-280).
    """

    @staticmethod
    def forward(ctx, diag, cvec, solver, x_init, U_warm, stats_sink):
        # the solve runs in the solver's precision (MpcSolver(dtype=...): float32 by default,
        # float64 = the reference's precision, policy.py:235-236); u0 comes back in diag's dtype
        ws, iterations, converged, _, _ = solver.solve_diag(x_init, diag.detach(), cvec.detach(), U_warm,
                                                            dtype=solver.dtype)
        ctx.solver = solver
        ctx.ws = ws
        ctx.out_dtype = diag.dtype
        ctx.out_device = diag.device
        if stats_sink is not None:
            stats_sink.setdefault("solves", 0)
            stats_sink.setdefault("non_converged", 0)
            stats_sink.setdefault("iterations", 0)
            # device-side counters (no host sync per solve); int() them when reading
            stats_sink["solves"] += ws.B
            stats_sink["non_converged"] = stats_sink["non_converged"] + (~converged).sum()
            stats_sink["iterations"] = stats_sink["iterations"] + iterations.sum()
        return ws.U[:, 0].to(device=diag.device, dtype=diag.dtype)

    @staticmethod
    def backward(ctx, grad_u0):
        ws, solver = ctx.ws, ctx.solver
        B, T, m = ws.U.shape
        seed = torch.zeros((B, T, m), dtype=ws.U.dtype, device=ws.U.device)
        seed[:, 0] = grad_u0.to(device=ws.U.device, dtype=ws.U.dtype)
        g = _solver.backward_raw(solver.model, solver.settings, ws.C, ws.c, ws.X, ws.U, None, seed,
                                 dtype=ws.U.dtype, device=ws.U.device)
        gd = g.dC.to(device=ctx.out_device, dtype=ctx.out_dtype)
        gc = g.dc.to(device=ctx.out_device, dtype=ctx.out_dtype)
        return gd, gc, None, None, None, None


def mpc_control(bundle, obs_t, solver, x_init, U_warm, stats_sink=None):
    """Differentiable path obs -> cost params -> solver -> first control (policy.py:286-290).

    ``bundle.actor(obs)`` must return (diag, cvec) of shape (B, T, n_z) each.
    """
    diag, cvec = bundle.actor(obs_t)
    return MpcSolveLayer.apply(diag, cvec, solver, x_init, U_warm, stats_sink)

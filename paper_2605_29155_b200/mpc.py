"""``MPC(n_state, n_ctrl, T, u_lower, u_upper, ...)`` — the differentiable MPC module API that
BASELINE.json's north_star names (the mpc.pytorch interface: time-major tensors,
``forward(x_init, QuadCost(C, c), dx) -> (x, u, cost)``), running the B200 kernels with
THIS reference's solver semantics (the fixed step-size list
alphas, conv_tol on the relative cost decrease, projected-Newton box QP).

Gradients flow, by implicit differentiation of the converged solve, to
  * x_init, the cost C (dense or diagonal) and c            (reference semantics),
  * the dynamics parameters theta of ``dx``                  (SURVEY.md §8(a) NEW row),
  * and through the returned optimal cost (envelope terms)   (SURVEY.md §8(a) NEW row).

Shapes (time-major like mpc.pytorch): x_init (B,n); C (T,B,nz,nz), (T,B,nz) diagonal, or
without the batch dim to broadcast; c (T,B,nz) or (T,nz). Returns x (T,B,n) = x_0..x_{T-1}
(mpc.pytorch convention; x_T is available as ``MPC.last_terminal_state``), u (T,B,m) and the
total stage cost (B,). There is no terminal cost term.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch
from torch import nn

from . import solver as _solver
from .dynamics import DynModel
from .errors import ConfigError, NumericError
from .settings import DEFAULT_ALPHAS, SolveSettings


class QuadCost(NamedTuple):
    C: torch.Tensor
    c: torch.Tensor


# ---------------------------------------------------------------------------- dynamics
class _Dx(nn.Module):
    """A dynamics module: a DynModel descriptor plus a differentiable parameter vector."""

    def __init__(self, model: DynModel, params=None, learn=False):
        super().__init__()
        self.template = model
        p = torch.as_tensor(model.params if params is None else params, dtype=torch.float64)
        if learn:
            self.params = nn.Parameter(p)
        else:
            self.register_buffer("params", p)

    @property
    def n_state(self):
        return self.template.n_x

    @property
    def n_ctrl(self):
        return self.template.n_u


class QuadrotorDx(_Dx):
    """13-state / 4-rotor quadrotor, params [m, arm, Jx, Jy, Jz, kappa, g]."""

    def __init__(self, dt=0.05, params=None, learn=False):
        super().__init__(DynModel.quadrotor(dt=dt), params, learn)


class PlanarQuadrotorDx(_Dx):
    """Planar quadrotor (6/2), params [m, arm, inertia, g] (dynamics.py:57-70)."""

    def __init__(self, dt=0.05, params=None, learn=False):
        super().__init__(DynModel.planar_quadrotor(dt=dt), params, learn)


class DoubleIntegratorDx(_Dx):
    def __init__(self, dim, dt):
        super().__init__(DynModel.double_integrator(dim, dt), None, False)


class LinDx(_Dx):
    """Time-invariant linear dynamics x+ = A x + B u, params = [A row-major, B row-major]."""

    def __init__(self, A, B, learn=False):
        A = torch.as_tensor(A, dtype=torch.float64)
        B = torch.as_tensor(B, dtype=torch.float64)
        model = DynModel.linear(A.detach().cpu().numpy(), B.detach().cpu().numpy())
        super().__init__(model, torch.cat([A.reshape(-1), B.reshape(-1)]), learn)


# ---------------------------------------------------------------------------- autograd
class _MPCFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x_init, C, c, theta, U_warm, model, settings, dtype, mpc):
        out = _solver.solve_raw(model, settings, x_init.detach(), C.detach(), c.detach(), U_warm,
                                dtype=dtype, theta=theta.detach(), device=x_init.device)
        ctx.model, ctx.settings, ctx.dtype, ctx.out = model, settings, dtype, out
        ctx.theta = theta.detach()
        ctx.in_dtype = x_init.dtype
        mpc._last = out
        return out.X, out.U, out.J

    @staticmethod
    def backward(ctx, gX, gU, gJ):
        out = ctx.out
        g = _solver.backward_raw(ctx.model, ctx.settings, out.C, out.c, out.X, out.U, gX, gU, gJ,
                                 dtype=ctx.dtype, theta=ctx.theta, want_theta=ctx.model.n_theta > 0,
                                 device=out.X.device)
        dth = g.dtheta.sum(0) if g.dtheta is not None else torch.zeros_like(ctx.theta)
        cast = lambda t: t.to(ctx.in_dtype)  # noqa: E731
        return cast(g.dx0), cast(g.dC), cast(g.dc), dth.to(ctx.theta.dtype), None, None, None, None, None


class MPC(nn.Module):
    """Differentiable box-constrained iLQR MPC layer (mpc.pytorch-style constructor)."""

    def __init__(self, n_state, n_ctrl, T, u_lower=None, u_upper=None, u_init=None, lqr_iter=10,
                 eps=1e-6, n_batch=None, alphas=DEFAULT_ALPHAS, boxqp_max_iter=20, boxqp_tol=1e-9,
                 exit_unconverged=False, detach_unconverged=False, backprop=True, verbose=0,
                 dtype=None, slew_rate_penalty=None, **_ignored):
        super().__init__()
        if slew_rate_penalty is not None:
            raise ConfigError("slew_rate_penalty is not part of the reference's cost model")
        self.n_state, self.n_ctrl, self.T = n_state, n_ctrl, T
        self.u_lower = self._bound(u_lower, -1e9)
        self.u_upper = self._bound(u_upper, 1e9)
        self.u_init = u_init
        self.settings = SolveSettings(T=T, u_min=self.u_lower, u_max=self.u_upper, K_max=lqr_iter,
                                      alphas=tuple(alphas), conv_tol=eps, boxqp_max_iter=boxqp_max_iter,
                                      boxqp_tol=boxqp_tol)
        self.exit_unconverged = exit_unconverged
        self.detach_unconverged = detach_unconverged
        self.backprop = backprop
        self.verbose = verbose
        self.dtype = dtype
        self._last = None

    def _bound(self, b, default):
        if b is None:
            return np.full(self.n_ctrl, default)
        t = b.detach().cpu().numpy() if isinstance(b, torch.Tensor) else np.asarray(b, dtype=np.float64)
        t = np.asarray(t, dtype=np.float64)
        if t.ndim == 0:
            return np.full(self.n_ctrl, float(t))
        flat = t.reshape(-1, self.n_ctrl)
        if not np.all(flat == flat[0]):
            raise ConfigError("time- or batch-varying control bounds are not supported (SolveSettings bounds)")
        return flat[0].copy()

    @property
    def last_terminal_state(self):
        return None if self._last is None else self._last.X[:, -1]

    @property
    def last_result(self):
        """The device-resident SolveOutput of the last forward (iterations, masks, gains...)."""
        return self._last

    def forward(self, x_init, cost: QuadCost, dx: _Dx):
        if dx.n_state != self.n_state or dx.n_ctrl != self.n_ctrl:
            raise ConfigError("dynamics dimensions do not match the MPC module")
        dev = x_init.device if x_init.is_cuda else _solver._device(None)
        dtype = self.dtype or (torch.float64 if x_init.dtype == torch.float64 else torch.float32)
        x_init = x_init.to(dev)
        B = x_init.shape[0]
        T, nz = self.T, self.n_state + self.n_ctrl
        C, c = cost
        C = torch.as_tensor(C, device=dev)
        c = torch.as_tensor(c, device=dev)
        # dense: (T,B,nz,nz) or (T,nz,nz); diagonal: (T,B,nz) or (T,nz). A 3-D tensor that
        # matches both readings (B == nz) is taken as the batched diagonal.
        if C.dim() == 4:
            diag = False
        elif C.dim() == 2:
            diag = True
            C = C[:, None].expand(T, B, nz)
        elif C.dim() == 3 and tuple(C.shape) == (T, B, nz):
            diag = True
        elif C.dim() == 3 and tuple(C.shape) == (T, nz, nz):
            diag = False
            C = C[:, None].expand(T, B, nz, nz)
        else:
            raise ConfigError(f"cost C has unsupported shape {tuple(C.shape)}")
        if tuple(C.shape[:2]) != (T, B):
            raise ConfigError(f"cost C must be time-major (T={T}, B={B}, ...), got {tuple(C.shape)}")
        if c.dim() == 2:
            c = c[:, None].expand(T, B, nz)
        Cb = C.transpose(0, 1).contiguous()  # time-major -> batch-major, once at the boundary
        cb = c.transpose(0, 1).contiguous()
        if self.u_init is None:
            u_h = np.clip(dx.template.hover_control(), self.u_lower, self.u_upper)
            U_warm = torch.as_tensor(u_h, device=dev, dtype=dtype).expand(B, T, self.n_ctrl).contiguous()
        else:
            U_warm = torch.as_tensor(self.u_init, device=dev).transpose(0, 1).contiguous()
        theta = dx.params.to(dev)
        model = dx.template
        if not self.backprop:
            with torch.no_grad():
                X, U, J = _MPCFunction.apply(x_init, Cb, cb, theta, U_warm, model, self.settings, dtype, self)
        else:
            X, U, J = _MPCFunction.apply(x_init, Cb, cb, theta, U_warm, model, self.settings, dtype, self)
        out = self._last
        if self.exit_unconverged and not bool(out.converged.all()):
            raise NumericError("some MPC instances did not converge within lqr_iter iterations")
        if self.detach_unconverged:
            keep = out.converged.to(X.dtype)
            X = X * keep[:, None, None] + (X * (1 - keep[:, None, None])).detach()
            U = U * keep[:, None, None] + (U * (1 - keep[:, None, None])).detach()
            J = J * keep + (J * (1 - keep)).detach()
        x = X[:, :T].transpose(0, 1).to(x_init.dtype)
        u = U.transpose(0, 1).to(x_init.dtype)
        return x, u, J.to(x_init.dtype)

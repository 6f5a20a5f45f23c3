"""The AC-MPC policy around the DiffMPC layer: a neural cost map (actor), a value head
(critic) and a learned exploration scale, plus the single-observation deployment step
``act``. API-compatible with /root/reference/pkg/src/fusedmpc/policy.py:37-174 and
:286-366 — same constructor arguments, parameter names and shapes (``actor.net.*``,
``critic.net.*``, ``log_sigma``), so a reference checkpoint's tensors load unchanged — but
the networks are GPU plumbing here: the hot path is the DiffMPC solve they feed
(``layer.MpcSolveLayer``), everything else is a few cuBLAS GEMMs.

Cost head (policy.py:93-110): sigmoid(net(obs)) reshaped to (T, 2, n_z) and mapped affinely
into [diag_lo, diag_hi] (diagonal of C_t) and [c_lo, c_hi] (c_t); the diagonal lower bound
keeps every C_t positive definite without a runtime regulariser (EPS_REG, qcost.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
from torch import nn

from .dynamics import DynModel
from .errors import ConfigError, NumericError
from .qcost import EPS_REG
from .settings import SolveSettings

LOG_2PI = math.log(2.0 * math.pi)


def _f64(a):
    return np.asarray(a, dtype=np.float64)


@dataclass(frozen=True)
class CostHeadScaling:
    """Per-entry affine ranges of the cost head: diag in [diag_lo, diag_hi], c in [c_lo, c_hi]
    (policy.py:45-80: diag_lo >= EPS_REG, upper bounds above lower bounds)."""

    diag_lo: np.ndarray
    diag_hi: np.ndarray
    c_lo: np.ndarray
    c_hi: np.ndarray

    def __post_init__(self):
        lo, hi, clo, chi = (_f64(getattr(self, k)) for k in ("diag_lo", "diag_hi", "c_lo", "c_hi"))
        for k, v in zip(("diag_lo", "diag_hi", "c_lo", "c_hi"), (lo, hi, clo, chi)):
            object.__setattr__(self, k, v)
        if (lo < EPS_REG).any():
            raise ConfigError(f"diagonal lower bounds must be >= {EPS_REG}")
        if (hi <= lo).any() or (chi <= clo).any():
            raise ConfigError("upper scaling bounds must exceed lower bounds")

    @staticmethod
    def default(n_z, diag_lo=1e-3, diag_hi=10.0, c_lo=-10.0, c_hi=10.0) -> "CostHeadScaling":
        full = lambda v: np.full(n_z, float(v))  # noqa: E731
        return CostHeadScaling(full(diag_lo), full(diag_hi), full(c_lo), full(c_hi))

    @staticmethod
    def for_model(model: DynModel, n_x: int, diag_lo=1e-3, diag_hi=10.0, c_lo=-10.0,
                  c_hi=10.0) -> "CostHeadScaling":
        """The control entries' c range is centred on -mean(diag) * u_rest, so an untrained
        (output 1/2) actor's cost is minimised at the rest control (hover), not at zero."""
        s = CostHeadScaling.default(n_x + model.n_u, diag_lo, diag_hi, c_lo, c_hi)
        shift = np.zeros(n_x + model.n_u)
        shift[n_x:] = -0.5 * (diag_lo + diag_hi) * model.hover_control()
        return CostHeadScaling(s.diag_lo, s.diag_hi, s.c_lo + shift, s.c_hi + shift)


def _mlp(widths) -> nn.Sequential:
    """Linear layers over consecutive widths with ReLU between them (none after the last)."""
    mods = []
    for k, (a, b) in enumerate(zip(widths[:-1], widths[1:])):
        if k:
            mods.append(nn.ReLU())
        mods.append(nn.Linear(a, b))
    return nn.Sequential(*mods)


class _Head(nn.Module):
    """An MLP followed by a fixed output map; ``kind`` selects the map:
    "cost" -> (diag, c) of shape (B, T, n_z) each, "action" -> bounded control mean,
    "value" -> scalar value."""

    def __init__(self, kind, obs_dim, hidden, out_dim, **bounds):
        super().__init__()
        self.kind = kind
        self.net = _mlp([obs_dim, *hidden, out_dim])
        self.shape = bounds.pop("shape", None)
        for k, v in bounds.items():
            self.register_buffer(k, torch.tensor(_f64(v), dtype=torch.float32))

    def forward(self, obs):
        y = self.net(obs)
        if self.kind == "value":
            return y.squeeze(-1)
        s = torch.sigmoid(y)
        if self.kind == "action":
            return self.u_lo + s * (self.u_hi - self.u_lo)
        s = s.view(-1, *self.shape)  # (B, T, 2, n_z): [diag | c] per stage
        return (self.diag_lo + s[:, :, 0] * (self.diag_hi - self.diag_lo),
                self.c_lo + s[:, :, 1] * (self.c_hi - self.c_lo))


def CostActor(obs_dim, T, n_z, scaling: CostHeadScaling, hidden=(512, 512)) -> nn.Module:
    """Observation -> per-stage (diag C_t, c_t) within the scaling bounds (policy.py:93-110)."""
    return _Head("cost", obs_dim, hidden, T * 2 * n_z, shape=(T, 2, n_z), diag_lo=scaling.diag_lo,
                 diag_hi=scaling.diag_hi, c_lo=scaling.c_lo, c_hi=scaling.c_hi)


def DirectActor(obs_dim, n_u, u_min, u_max, hidden=(512, 512)) -> nn.Module:
    """Observation -> control mean in [u_min, u_max] (the solver-free ac_mlp head)."""
    return _Head("action", obs_dim, hidden, n_u, u_lo=u_min, u_hi=u_max)


def Critic(obs_dim, hidden=(512, 512)) -> nn.Module:
    return _Head("value", obs_dim, hidden, 1)


class PolicyBundle(nn.Module):
    """Actor + critic + log exploration scale (policy.py:136-174; same arguments). The
    initial scale is sigma_init_scale * (u_max - u_min) per control."""

    def __init__(self, mode, obs_dim, model: DynModel, settings: SolveSettings, scaling: CostHeadScaling,
                 hidden=(512, 512), sigma_init_scale=0.1):
        super().__init__()
        if mode not in ("ac_mpc", "ac_mlp"):
            raise ConfigError(f"policy mode must be ac_mpc or ac_mlp, got {mode!r}")
        u_min, u_max = settings.bounds_for(model.n_u)
        self.mode, self.obs_dim, self.T, self.hidden = mode, obs_dim, settings.T, tuple(hidden)
        self.n_x, self.n_u, self.n_z = model.n_x, model.n_u, model.n_x + model.n_u
        self.u_min, self.u_max = u_min, u_max
        self.scaling, self.sigma_init_scale = scaling, sigma_init_scale
        if mode == "ac_mpc":
            self.actor = CostActor(obs_dim, settings.T, self.n_z, scaling, hidden)
        else:
            self.actor = DirectActor(obs_dim, model.n_u, u_min, u_max, hidden)
        self.critic = Critic(obs_dim, hidden)
        self.log_sigma = nn.Parameter(torch.tensor(np.log(sigma_init_scale * (u_max - u_min)),
                                                   dtype=torch.float32))

    def sigma(self) -> np.ndarray:
        return np.exp(self.log_sigma.detach().double().cpu().numpy())


# --------------------------------------------------------------------------- deployment
@dataclass
class PolicyAction:
    """One policy step (policy.py:179-186)."""

    u_mpc: np.ndarray
    u_sampled: np.ndarray   # executed control, clamped to the bounds
    log_prob: float         # Gaussian density of the PRE-clamp sample
    sigma: np.ndarray
    u_raw: np.ndarray = None


def gaussian_log_prob(x, mean, sigma) -> float:
    z = (_f64(x) - mean) / sigma
    return float(np.sum(-0.5 * z * z - np.log(sigma) - 0.5 * LOG_2PI))


def _obs_tensor(bundle, obs):
    obs = _f64(obs)
    if obs.shape != (bundle.obs_dim,):
        raise ConfigError(f"obs has shape {obs.shape}, expected ({bundle.obs_dim},)")
    if not np.isfinite(obs).all():
        raise NumericError("non-finite observation")
    dev = next(bundle.parameters()).device
    return torch.tensor(obs, dtype=torch.float32, device=dev)[None]


def actor_forward(bundle: PolicyBundle, obs):
    """One observation -> StageCostParams.from_diag of the actor's output (policy.py:293-309)."""
    from .qcost import StageCostParams

    if bundle.mode != "ac_mpc":
        raise ConfigError("actor_forward requires an ac_mpc bundle")
    with torch.no_grad():
        diag, cvec = bundle.actor(_obs_tensor(bundle, obs))
    diag, cvec = diag[0].double().cpu().numpy(), cvec[0].double().cpu().numpy()
    if not (np.isfinite(diag).all() and np.isfinite(cvec).all()):
        raise NumericError("non-finite actor output")
    return StageCostParams.from_diag(diag, cvec, bundle.n_x)


def critic_forward(bundle: PolicyBundle, obs):
    """Scalar value for one observation, a vector for a batch (policy.py:312-321)."""
    obs = _f64(obs)
    dev = next(bundle.parameters()).device
    with torch.no_grad():
        v = bundle.critic(torch.tensor(np.atleast_2d(obs), dtype=torch.float32, device=dev))
    v = v.double().cpu().numpy()
    if not np.isfinite(v).all():
        raise NumericError("non-finite critic output")
    return float(v[0]) if obs.ndim == 1 else v


def act(bundle: PolicyBundle, obs, x_init, solver, explore: bool, rng: np.random.Generator, slot: int = 0,
        U_warm=None) -> PolicyAction:
    """Deployment step, B = 1 (policy.py:324-366): actor -> StageCostParams.from_diag (the
    object path's symmetrisation / C_uu regularisation) -> one DiffMPC solve on the GPU
    (latency kernel) warm-started from the solver's slot -> first control; the solution is
    pushed back as the slot's shifted warm start. With ``explore`` the executed control is a
    clamped Gaussian sample around it and ``log_prob`` is the pre-clamp sample's density.
    Raises NumericError when the solve fails (reference semantics)."""
    sigma = bundle.sigma()
    if bundle.mode == "ac_mpc":
        p = actor_forward(bundle, obs)
        U0 = solver.warm[slot] if U_warm is None else U_warm
        U0 = torch.as_tensor(U0, dtype=torch.float64).reshape(1, bundle.T, bundle.n_u)
        diag = np.diagonal(p.C, axis1=1, axis2=2)  # the regularised diagonal (policy.py:343-348)
        ws, _, _, _, _ = solver.solve_diag(_f64(x_init)[None], diag[None], p.c[None], U0, dtype=torch.float64)
        if bool(ws.failed[0]):
            raise NumericError(f"solver failed during act (slot {slot})")
        u_mpc = ws.U[0, 0].double().cpu().numpy()
        solver.push_warm(ws.U, slots=[slot])
    else:
        with torch.no_grad():
            u_mpc = bundle.actor(_obs_tensor(bundle, obs))[0].double().cpu().numpy()
    u_raw = rng.normal(u_mpc, sigma) if explore else u_mpc.copy()
    return PolicyAction(u_mpc=u_mpc, u_sampled=np.clip(u_raw, bundle.u_min, bundle.u_max) if explore else u_mpc.copy(),
                        log_prob=gaussian_log_prob(u_raw, u_mpc, sigma), sigma=sigma, u_raw=u_raw)

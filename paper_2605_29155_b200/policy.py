"""Actor / critic networks around the differentiable solver (the AC-MPC policy), mirroring
/root/reference/pkg/src/fusedmpc/policy.py:37-174 so a reference checkpoint's layer shapes
and the cost-head squashing carry over unchanged.

The actor is a neural cost map: observation -> per-timestep diagonal cost (diag C_t, c_t),
squashed by a sigmoid into configured bounds (policy.py:93-110). Its output feeds
``layer.MpcSolveLayer`` on the GPU; the networks themselves are plain torch modules
(cuBLAS GEMMs: the DiffMPC layer is the hot path, the 2x512 MLPs are plumbing).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
from torch import nn

from .dynamics import DynModel
from .errors import ConfigError
from .qcost import EPS_REG
from .settings import SolveSettings

LOG_2PI = math.log(2.0 * math.pi)


@dataclass(frozen=True)
class MlpSpec:
    """Layer widths and output head of a policy network (policy.py:37-42)."""

    hidden: tuple = (512, 512)
    head: str = "cost"


@dataclass(frozen=True)
class CostHeadScaling:
    """Bounds mapping sigmoid outputs to cost coefficients (policy.py:45-80)."""

    diag_lo: np.ndarray
    diag_hi: np.ndarray
    c_lo: np.ndarray
    c_hi: np.ndarray

    def __post_init__(self):
        for name in ("diag_lo", "diag_hi", "c_lo", "c_hi"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        if np.any(self.diag_lo < EPS_REG):
            raise ConfigError(f"diagonal lower bounds must be >= {EPS_REG}")
        if np.any(self.diag_hi <= self.diag_lo) or np.any(self.c_hi <= self.c_lo):
            raise ConfigError("upper scaling bounds must exceed lower bounds")

    @staticmethod
    def default(n_z, diag_lo=1e-3, diag_hi=10.0, c_lo=-10.0, c_hi=10.0) -> "CostHeadScaling":
        return CostHeadScaling(np.full(n_z, diag_lo), np.full(n_z, diag_hi), np.full(n_z, c_lo),
                               np.full(n_z, c_hi))

    @staticmethod
    def for_model(model: DynModel, n_x: int, diag_lo=1e-3, diag_hi=10.0, c_lo=-10.0,
                  c_hi=10.0) -> "CostHeadScaling":
        """Control-dim linear range shifted so its midpoint encodes the rest control
        (policy.py:66-80): a zero-initialised actor regulates toward hover."""
        n_z = n_x + model.n_u
        s = CostHeadScaling.default(n_z, diag_lo, diag_hi, c_lo, c_hi)
        offset = -0.5 * (diag_lo + diag_hi) * model.hover_control()
        c_lo_arr, c_hi_arr = s.c_lo.copy(), s.c_hi.copy()
        c_lo_arr[n_x:] += offset
        c_hi_arr[n_x:] += offset
        return CostHeadScaling(s.diag_lo, s.diag_hi, c_lo_arr, c_hi_arr)


def build_mlp(in_dim, hidden, out_dim):
    layers, last = [], in_dim
    for width in hidden:
        layers += [nn.Linear(last, width), nn.ReLU()]
        last = width
    layers.append(nn.Linear(last, out_dim))
    return nn.Sequential(*layers)


class CostActor(nn.Module):
    """Observation -> per-timestep (diag C_t, c_t) within scaling bounds (policy.py:93-110)."""

    def __init__(self, obs_dim, T, n_z, scaling: CostHeadScaling, hidden=(512, 512)):
        super().__init__()
        self.T, self.n_z = T, n_z
        self.net = build_mlp(obs_dim, hidden, T * 2 * n_z)
        for name in ("diag_lo", "diag_hi", "c_lo", "c_hi"):
            self.register_buffer(name, torch.tensor(getattr(scaling, name), dtype=torch.float32))

    def forward(self, obs):
        raw = torch.sigmoid(self.net(obs)).view(-1, self.T, 2, self.n_z)
        diag = self.diag_lo + raw[:, :, 0, :] * (self.diag_hi - self.diag_lo)
        cvec = self.c_lo + raw[:, :, 1, :] * (self.c_hi - self.c_lo)
        return diag, cvec


class DirectActor(nn.Module):
    """Observation -> control mean within bounds (the solver-free baseline, policy.py:113-124)."""

    def __init__(self, obs_dim, n_u, u_min, u_max, hidden=(512, 512)):
        super().__init__()
        self.net = build_mlp(obs_dim, hidden, n_u)
        self.register_buffer("u_lo", torch.tensor(u_min, dtype=torch.float32))
        self.register_buffer("u_hi", torch.tensor(u_max, dtype=torch.float32))

    def forward(self, obs):
        return self.u_lo + torch.sigmoid(self.net(obs)) * (self.u_hi - self.u_lo)


class Critic(nn.Module):
    def __init__(self, obs_dim, hidden=(512, 512)):
        super().__init__()
        self.net = build_mlp(obs_dim, hidden, 1)

    def forward(self, obs):
        return self.net(obs).squeeze(-1)


class PolicyBundle(nn.Module):
    """Actor + critic + exploration std (policy.py:136-174)."""

    def __init__(self, mode, obs_dim, model: DynModel, settings: SolveSettings, scaling: CostHeadScaling,
                 hidden=(512, 512), sigma_init_scale=0.1):
        super().__init__()
        if mode not in ("ac_mpc", "ac_mlp"):
            raise ConfigError(f"policy mode must be ac_mpc or ac_mlp, got {mode!r}")
        self.mode, self.obs_dim, self.T = mode, obs_dim, settings.T
        self.n_x, self.n_u = model.n_x, model.n_u
        self.n_z = model.n_x + model.n_u
        self.hidden = tuple(hidden)
        self.scaling = scaling
        self.sigma_init_scale = sigma_init_scale
        u_min, u_max = settings.bounds_for(model.n_u)
        self.u_min, self.u_max = u_min, u_max
        if mode == "ac_mpc":
            self.actor_spec = MlpSpec(self.hidden, head="cost")
            self.actor = CostActor(obs_dim, settings.T, self.n_z, scaling, hidden)
        else:
            self.actor_spec = MlpSpec(self.hidden, head="action")
            self.actor = DirectActor(obs_dim, model.n_u, u_min, u_max, hidden)
        self.critic_spec = MlpSpec(self.hidden, head="value")
        self.critic = Critic(obs_dim, hidden)
        sigma0 = sigma_init_scale * (u_max - u_min)
        self.log_sigma = nn.Parameter(torch.tensor(np.log(sigma0), dtype=torch.float32))

    def sigma(self) -> np.ndarray:
        return np.exp(self.log_sigma.detach().cpu().numpy().astype(np.float64))

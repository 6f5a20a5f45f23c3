"""Batched planar gate-racing environment, stepped on the GPU.

Semantics follow /root/reference/pkg/src/fusedmpc/raceenv.py per environment: gates are
segments of a given width centred on ``center`` and perpendicular to the unit ``normal``;
passing = crossing the gate plane in the normal direction within half a width of the
centre (boundary inclusive); crossing within ``miss_factor`` half-widths is a terminal
miss; shaped progress reward toward the next gate, gate bonus, crash / time penalties,
timeout (raceenv.py:174-228). The observation (11 values, raceenv.py:120-140) and the
MPC state (drone state translated to the next gate, raceenv.py:143-149) are the
reference's.

B200 design: the N environments live in device tensors (state (N,6) float64, gate index,
lap count, episode time, done flags); one ``step`` advances all of them with the drone
dynamics evaluated by the library's CUDA dynamics kernel (``diffmpc_dynamics_f64``, the
same model code the iLQR kernels use) and the gate / reward logic as batched tensor ops —
no host round trip, so rollout collection stays on the device. Random spawn perturbations
come from a device ``torch.Generator`` (the reference draws per-env numpy streams; the
distributions match, the streams do not).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .dynamics import DynModel
from .errors import ConfigError

OBS_DIM = 11
POS_SCALE = 0.2
VEL_SCALE = 0.2
OMEGA_SCALE = 0.2

# termination reasons (raceenv.py:35-38), as integer codes
REASON_NONE, REASON_LAP, REASON_MISS, REASON_OOB, REASON_TIMEOUT = 0, 1, 2, 3, 4
REASON_NAMES = {REASON_NONE: "", REASON_LAP: "lap_complete", REASON_MISS: "gate_missed",
                REASON_OOB: "out_of_bounds", REASON_TIMEOUT: "timeout"}


@dataclass(frozen=True)
class Gate:
    center: np.ndarray
    normal: np.ndarray
    width: float

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=np.float64))
        object.__setattr__(self, "normal", np.asarray(self.normal, dtype=np.float64))
        if self.width <= 0.0:
            raise ConfigError(f"gate width must be positive, got {self.width}")
        if abs(np.linalg.norm(self.normal) - 1.0) > 1e-9:
            raise ConfigError("gate normal must be unit length (tolerance 1e-9)")


@dataclass(frozen=True)
class TrackSpec:
    gates: tuple
    laps: int
    spawn: np.ndarray
    margin: float = 5.0

    def __post_init__(self):
        object.__setattr__(self, "gates", tuple(self.gates))
        object.__setattr__(self, "spawn", np.asarray(self.spawn, dtype=np.float64))
        if len(self.gates) < 2:
            raise ConfigError("a track needs at least 2 gates")
        if self.laps < 1:
            raise ConfigError("laps must be >= 1")
        pts = np.array([g.center for g in self.gates] + [self.spawn[:2]])
        object.__setattr__(self, "lo", pts.min(axis=0) - self.margin)
        object.__setattr__(self, "hi", pts.max(axis=0) + self.margin)


def load_track(path) -> TrackSpec:
    """Read a track file (YAML: spawn, laps, gates with center / normal / width)."""
    import yaml

    with open(path) as f:
        raw = yaml.safe_load(f)
    try:
        gates = [Gate(np.array(g["center"]), np.array(g["normal"]), float(g["width"])) for g in raw["gates"]]
        return TrackSpec(gates=gates, laps=int(raw.get("laps", 1)), spawn=np.array(raw["spawn"], dtype=np.float64))
    except (KeyError, TypeError) as e:
        raise ConfigError(f"malformed track file {path}: {e}") from e


def hairpin5() -> TrackSpec:
    """The reference's bundled 5-gate track with a reversal after gate 3 (tracks/hairpin5.yaml)."""
    r = float(np.sqrt(0.5))
    g = [((3.0, 0.0), (1.0, 0.0)), ((7.0, 2.0), (r, r)), ((9.0, 6.0), (0.0, 1.0)),
         ((6.0, 9.0), (-1.0, 0.0)), ((1.0, 6.0), (-r, -r))]
    return TrackSpec(gates=[Gate(np.array(c), np.array(n), 3.0) for c, n in g], laps=1, spawn=np.zeros(6))


@dataclass(frozen=True)
class RewardConfig:
    """raceenv.py:88-99 (same defaults)."""

    k_p: float = 1.0
    gate_bonus: float = 10.0
    crash_penalty: float = 10.0
    time_penalty: float = 0.1
    progress_cap: float = 5.0
    timeout: float = 20.0
    miss_factor: float = 2.0


class BatchedRaceEnv:
    """N environments on one device; ``step`` advances all of them at once."""

    def __init__(self, track: TrackSpec, model: DynModel, n_envs: int, cfg: RewardConfig = RewardConfig(),
                 device=None, seed: int = 0, reset_noise: float = 0.1):
        if model.n_x != 6 or model.n_u != 2:
            raise ConfigError("the race environment is planar (6 states, 2 rotors)")
        self.track, self.model, self.cfg, self.N = track, model, cfg, int(n_envs)
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.reset_noise = float(reset_noise)
        f = dict(dtype=torch.float64, device=self.device)
        self.centers = torch.tensor(np.stack([g.center for g in track.gates]), **f)
        self.normals = torch.tensor(np.stack([g.normal for g in track.gates]), **f)
        self.widths = torch.tensor([g.width for g in track.gates], **f)
        self.lo = torch.tensor(track.lo, **f)
        self.hi = torch.tensor(track.hi, **f)
        self.spawn = torch.tensor(track.spawn, **f)
        self.n_gates = len(track.gates)
        self.gen = torch.Generator(device=self.device).manual_seed(seed)
        self.x = self.spawn.expand(self.N, 6).clone()
        self.gate = torch.zeros(self.N, dtype=torch.int64, device=self.device)
        self.laps = torch.zeros_like(self.gate)
        self.t = torch.zeros(self.N, **f)
        self.done = torch.zeros(self.N, dtype=torch.bool, device=self.device)
        self.reason = torch.zeros(self.N, dtype=torch.int64, device=self.device)
        self.obs_dim = OBS_DIM

    # --------------------------------------------------------------- queries
    def observation(self) -> torch.Tensor:
        """(N, 11) float64 (raceenv.py:120-140)."""
        x = self.x
        g1 = self.gate
        g2 = (g1 + 1) % self.n_gates
        c1, n1, c2 = self.centers[g1], self.normals[g1], self.centers[g2]
        return torch.stack([
            (c1[:, 0] - x[:, 0]) * POS_SCALE, (c1[:, 1] - x[:, 1]) * POS_SCALE, n1[:, 0], n1[:, 1],
            (c2[:, 0] - x[:, 0]) * POS_SCALE, (c2[:, 1] - x[:, 1]) * POS_SCALE,
            x[:, 3] * VEL_SCALE, x[:, 4] * VEL_SCALE, torch.sin(x[:, 2]), torch.cos(x[:, 2]),
            x[:, 5] * OMEGA_SCALE], dim=1)

    def mpc_state(self) -> torch.Tensor:
        """Drone state translated so the next gate centre is the origin (raceenv.py:143-149)."""
        x = self.x.clone()
        x[:, 0:2] -= self.centers[self.gate]
        return x

    # --------------------------------------------------------------- dynamics
    def reset(self, mask: torch.Tensor | None = None) -> torch.Tensor:
        """Respawn the masked environments (all if None) with the Gaussian position
        perturbation of raceenv.py:152-158; returns the full observation."""
        m = torch.ones(self.N, dtype=torch.bool, device=self.device) if mask is None else mask
        x = self.spawn.expand(self.N, 6).clone()
        if self.reset_noise > 0.0:
            x[:, 0:2] += self.reset_noise * torch.randn((self.N, 2), generator=self.gen, dtype=torch.float64,
                                                        device=self.device)
        mm = m[:, None]
        self.x = torch.where(mm, x, self.x)
        self.gate = torch.where(m, 0, self.gate)
        self.laps = torch.where(m, 0, self.laps)
        self.t = torch.where(m, 0.0, self.t)
        self.done = torch.where(m, False, self.done)
        self.reason = torch.where(m, REASON_NONE, self.reason)
        return self.observation()

    def step(self, u: torch.Tensor):
        """Advance every environment one control period (raceenv.py:174-228).

        Returns (obs (N,11), reward (N,), done (N,), reason (N,)); environments that were
        already done are not advanced (the reference raises; callers reset them)."""
        from .solver import dynamics_t

        cfg = self.cfg
        live = ~self.done
        u = u.to(device=self.device, dtype=torch.float64)
        x_new, _, _ = dynamics_t(self.model, self.x, u, dtype=torch.float64, device=self.device)
        t_new = self.t + self.model.dt
        gi = self.gate
        c, n, w = self.centers[gi], self.normals[gi], self.widths[gi]
        p_prev, p_new = self.x[:, 0:2], x_new[:, 0:2]
        reward = torch.full((self.N,), -cfg.time_penalty * self.model.dt, dtype=torch.float64, device=self.device)
        finite = torch.isfinite(x_new).all(dim=1)
        x_new = torch.where(torch.isfinite(x_new), x_new, torch.zeros_like(x_new))
        # shaped progress
        d_prev = torch.linalg.vector_norm(p_prev - c, dim=1)
        d_new = torch.linalg.vector_norm(p_new - c, dim=1)
        reward = reward + torch.where(finite, torch.clamp(cfg.k_p * (d_prev - d_new), -cfg.progress_cap,
                                                          cfg.progress_cap), 0.0)
        # gate-plane crossing (raceenv.py:161-171)
        s_prev = ((p_prev - c) * n).sum(1)
        s_new = ((p_new - c) * n).sum(1)
        crossed = (s_prev <= 0.0) & (s_new > 0.0)
        denom = s_prev - s_new
        frac = torch.where(s_new != s_prev, s_prev / torch.where(denom == 0, 1.0, denom), 0.0)
        p_cross = p_prev + frac[:, None] * (p_new - p_prev)
        tang = torch.stack([-n[:, 1], n[:, 0]], dim=1)
        lateral = ((p_cross - c) * tang).sum(1).abs()
        hw = w / 2.0
        passed = finite & crossed & (lateral <= hw)
        missed = finite & crossed & ~passed & (lateral <= cfg.miss_factor * hw)
        inb = ((p_new >= self.lo) & (p_new <= self.hi)).all(dim=1)
        oob = ~finite | (finite & ~passed & ~missed & ~inb)
        reward = reward + torch.where(passed, cfg.gate_bonus, 0.0)
        nxt = self.gate + passed.to(torch.int64)
        wrap = nxt == self.n_gates
        laps = self.laps + wrap.to(torch.int64)
        nxt = torch.where(wrap, 0, nxt)
        lap_done = wrap & (laps >= self.track.laps)
        reward = reward - torch.where(missed | oob, cfg.crash_penalty, 0.0)
        done = lap_done | missed | oob
        timeout = ~done & (t_new >= cfg.timeout)
        done = done | timeout
        reason = torch.where(lap_done, REASON_LAP, torch.where(missed, REASON_MISS, torch.where(
            oob, REASON_OOB, torch.where(timeout, REASON_TIMEOUT, REASON_NONE))))
        # only live environments advance
        self.x = torch.where(live[:, None], x_new, self.x)
        self.t = torch.where(live, t_new, self.t)
        self.gate = torch.where(live, nxt, self.gate)
        self.laps = torch.where(live, laps, self.laps)
        self.reason = torch.where(live, reason, self.reason)
        reward = torch.where(live, reward, 0.0)
        self.done = self.done | (live & done)
        return self.observation(), reward, self.done.clone(), self.reason.clone()

"""Batched gate-racing environments, stepped on the GPU.

Planar (the reference's environment, /root/reference/pkg/src/fusedmpc/raceenv.py): gates are
segments of a given width centred on ``center`` and perpendicular to the unit ``normal``;
passing = crossing the gate plane in the normal direction within half a width of the centre
(boundary inclusive); crossing within ``miss_factor`` half-widths is a terminal miss; shaped
progress reward toward the next gate, gate bonus, crash / time penalties, timeout
(raceenv.py:174-228). Observation: 11 values (raceenv.py:120-140); MPC state: the drone
state translated so the next gate's centre is the origin (raceenv.py:143-149).

3-D (new; the 13-state quadrotor of BASELINE config 4, which the reference does not have):
the same rules with circular gate openings of diameter ``width`` (a crossing passes when the
crossing point lies within width/2 of the centre in the gate plane) and a 19-value
observation: [(g1 - p) * POS_SCALE (3), n1 (3), (g2 - p) * POS_SCALE (3), v * VEL_SCALE (3),
q (4, w x y z), omega * OMEGA_SCALE (3)].

B200 design: the N environments live in device tensors (state (N,nx) float64, gate index,
lap count, episode time, done flags) and ``step`` is ONE kernel launch
(``diffmpc_race_step_f64``, csrc/raceenv.cu: dynamics with the library's model code, gate
logic, reward, termination and the next observation per thread) — no host round trip, so
rollout collection stays on the device and is capturable in a CUDA graph. Random spawn
perturbations come from a device ``torch.Generator`` (the reference draws per-env numpy
streams; the distributions match, the streams do not).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .dynamics import DynModel
from .errors import ConfigError

OBS_DIM = 11       # planar observation (raceenv.py:120-140)
OBS_DIM_3D = 19    # 3-D observation (13-state quadrotor), see the module docstring
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
        dims = {len(g.center) for g in self.gates} | {len(g.normal) for g in self.gates}
        if len(dims) != 1 or dims.pop() not in (2, 3):
            raise ConfigError("gate centres and normals must all be 2-D (planar) or all 3-D")
        object.__setattr__(self, "dim", len(self.gates[0].center))
        pts = np.array([g.center for g in self.gates] + [self.spawn[:self.dim]])
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


def helix5() -> TrackSpec:
    """A 3-D counterpart of hairpin5 for the 13-state quadrotor: five 1.5 m-diameter gates on
    a climbing then descending loop, passed counter-clockwise; spawn at rest (hover
    attitude) 1 m above the ground level of the first gate."""
    gates = []
    for k in range(5):
        a = 2.0 * np.pi * k / 5.0
        c = np.array([6.0 * np.cos(a), 6.0 * np.sin(a), 2.0 + 1.0 * np.sin(a)])
        tang = np.array([-np.sin(a), np.cos(a), 1.0 * np.cos(a) / 6.0])  # d(c)/da, normalised
        gates.append(Gate(c, tang / np.linalg.norm(tang), 1.5))
    spawn = np.zeros(13)
    spawn[0:3] = [6.0, -3.0, 1.0]
    spawn[3] = 1.0
    return TrackSpec(gates=gates, laps=1, spawn=spawn)


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
    """N environments on one device; ``step`` advances all of them in one kernel launch.
    Planar quadrotor (6 states, 2 rotors) on a 2-D track, or the 13-state quadrotor on a 3-D
    track (e.g. ``helix5()``)."""

    def __init__(self, track: TrackSpec, model: DynModel, n_envs: int, cfg: RewardConfig = RewardConfig(),
                 device=None, seed: int = 0, reset_noise: float = 0.1):
        from . import _abi
        from .dynamics import KIND_PLANAR_QUADROTOR, KIND_QUADROTOR13

        if track.dim == 2 and model.kind == KIND_PLANAR_QUADROTOR:
            self.pos, self.vel, self.obs_dim = slice(0, 2), slice(3, 5), OBS_DIM
        elif track.dim == 3 and model.kind == KIND_QUADROTOR13:
            self.pos, self.vel, self.obs_dim = slice(0, 3), slice(7, 10), OBS_DIM_3D
        else:
            raise ConfigError("race environments: planar quadrotor on a 2-D track or the 13-state "
                              "quadrotor on a 3-D track")
        if len(track.spawn) != model.n_x:
            raise ConfigError(f"spawn state must have {model.n_x} entries")
        self.track, self.model, self.cfg, self.N = track, model, cfg, int(n_envs)
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.reset_noise = float(reset_noise)
        self.D = track.dim
        f = dict(dtype=torch.float64, device=self.device)
        self.centers = torch.tensor(np.stack([g.center for g in track.gates]), **f)
        self.normals = torch.tensor(np.stack([g.normal for g in track.gates]), **f)
        self.spawn = torch.tensor(track.spawn, **f)
        self.theta = torch.tensor(np.asarray(model.params, dtype=np.float64), **f)
        self.n_gates = len(track.gates)
        self._track = _abi.make_track(track, cfg, POS_SCALE, VEL_SCALE, OMEGA_SCALE)
        self.gen = torch.Generator(device=self.device).manual_seed(seed)
        self.x = self.spawn.expand(self.N, model.n_x).clone()
        self.gate = torch.zeros(self.N, dtype=torch.int64, device=self.device)
        self.laps = torch.zeros_like(self.gate)
        self.t = torch.zeros(self.N, **f)
        self.done = torch.zeros(self.N, dtype=torch.bool, device=self.device)
        self.reason = torch.zeros(self.N, dtype=torch.int64, device=self.device)

    # --------------------------------------------------------------- queries
    def observation(self) -> torch.Tensor:
        """(N, 11) planar (raceenv.py:120-140) or (N, 19) 3-D observation, float64."""
        x, D = self.x, self.D
        g1 = self.gate
        c1, n1, c2 = self.centers[g1], self.normals[g1], self.centers[(g1 + 1) % self.n_gates]
        p = x[:, self.pos]
        if D == 2:
            return torch.stack([
                (c1[:, 0] - p[:, 0]) * POS_SCALE, (c1[:, 1] - p[:, 1]) * POS_SCALE, n1[:, 0], n1[:, 1],
                (c2[:, 0] - p[:, 0]) * POS_SCALE, (c2[:, 1] - p[:, 1]) * POS_SCALE,
                x[:, 3] * VEL_SCALE, x[:, 4] * VEL_SCALE, torch.sin(x[:, 2]), torch.cos(x[:, 2]),
                x[:, 5] * OMEGA_SCALE], dim=1)
        return torch.cat([(c1 - p) * POS_SCALE, n1, (c2 - p) * POS_SCALE, x[:, self.vel] * VEL_SCALE,
                          x[:, 3:7], x[:, 10:13] * OMEGA_SCALE], dim=1)

    def mpc_state(self) -> torch.Tensor:
        """Drone state translated so the next gate centre is the origin (raceenv.py:143-149)."""
        x = self.x.clone()
        x[:, self.pos] -= self.centers[self.gate]
        return x

    # --------------------------------------------------------------- dynamics
    def reset(self, mask: torch.Tensor | None = None) -> torch.Tensor:
        """Respawn the masked environments (all if None) with the Gaussian position
        perturbation of raceenv.py:152-158; returns the full observation."""
        m = torch.ones(self.N, dtype=torch.bool, device=self.device) if mask is None else mask
        x = self.spawn.expand(self.N, self.model.n_x).clone()
        if self.reset_noise > 0.0:
            x[:, self.pos] += self.reset_noise * torch.randn((self.N, self.D), generator=self.gen,
                                                             dtype=torch.float64, device=self.device)
        self.x = torch.where(m[:, None], x, self.x)
        self.gate = torch.where(m, 0, self.gate)
        self.laps = torch.where(m, 0, self.laps)
        self.t = torch.where(m, 0.0, self.t)
        self.done = torch.where(m, False, self.done)
        self.reason = torch.where(m, REASON_NONE, self.reason)
        return self.observation()

    def step(self, u: torch.Tensor):
        """Advance every environment one control period (raceenv.py:174-228) in ONE kernel.

        Returns (obs (N, obs_dim), reward (N,), done (N,), reason (N,)); environments that
        were already done are not advanced (the reference raises; callers reset them)."""
        import ctypes

        from . import _lib
        from .solver import _stream

        u = u.to(device=self.device, dtype=torch.float64).contiguous()
        if tuple(u.shape) != (self.N, self.model.n_u):
            raise ConfigError(f"u must be ({self.N}, {self.model.n_u})")
        for name in ("x", "gate", "laps", "t", "done", "reason"):
            v = getattr(self, name)
            if not v.is_contiguous():
                setattr(self, name, v.contiguous())
        reward = torch.empty(self.N, dtype=torch.float64, device=self.device)
        obs = torch.empty((self.N, self.obs_dim), dtype=torch.float64, device=self.device)
        P = lambda t: t.data_ptr()  # noqa: E731
        _lib.check(_lib.lib().diffmpc_race_step_f64(
            ctypes.byref(self._track), int(self.model.kind), self.N, float(self.model.dt), P(self.theta),
            P(self.x), P(self.gate), P(self.laps), P(self.t), P(self.done), P(self.reason), P(u), P(reward), P(obs),
            _stream(None, self.device)))
        return obs, reward, self.done.clone(), self.reason.clone()

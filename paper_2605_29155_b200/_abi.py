"""ctypes mirror of include/diffmpc.h (the C ABI structs) and helpers that fill them
from a (DynModel, SolveSettings) pair. Pure host logic, no compute."""

from __future__ import annotations

import ctypes

import numpy as np

from .errors import ConfigError

MAX_NU = 8
MAX_ALPHA = 8
COST_DENSE = 0
COST_DIAG = 1
KERNEL_AUTO, KERNEL_THROUGHPUT, KERNEL_LATENCY = 0, 1, 2
_KERNELS = {"auto": KERNEL_AUTO, "throughput": KERNEL_THROUGHPUT, "latency": KERNEL_LATENCY}


def kernel_code(kernel) -> int:
    if isinstance(kernel, int) and kernel in _KERNELS.values():
        return kernel
    if kernel not in _KERNELS:
        raise ConfigError(f"kernel must be one of {tuple(_KERNELS)}, got {kernel!r}")
    return _KERNELS[kernel]
ABI_VERSION = 2


class DiffMPCProblem(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int32),
        ("T", ctypes.c_int32),
        ("nx", ctypes.c_int32),
        ("nu", ctypes.c_int32),
        ("model_kind", ctypes.c_int32),
        ("cost_layout", ctypes.c_int32),
        ("K_max", ctypes.c_int32),
        ("n_alpha", ctypes.c_int32),
        ("boxqp_max_iter", ctypes.c_int32),
        ("n_theta", ctypes.c_int32),
        ("theta_stride", ctypes.c_int32),
        ("kernel_select", ctypes.c_int32),
        ("dt", ctypes.c_double),
        ("conv_tol", ctypes.c_double),
        ("boxqp_tol", ctypes.c_double),
        ("u_min", ctypes.c_double * MAX_NU),
        ("u_max", ctypes.c_double * MAX_NU),
        ("alphas", ctypes.c_double * MAX_ALPHA),
    ]


_vp = ctypes.c_void_p


class DiffMPCForwardIO(ctypes.Structure):
    _fields_ = [(n, _vp) for n in (
        "theta", "C", "c", "x0", "U_warm", "X", "U", "J", "K", "k", "iters", "converged",
        "diverged", "fail_t", "clamped", "alpha_hist", "J_hist", "workspace")] + [
        ("workspace_bytes", ctypes.c_uint64)]


class DiffMPCBackwardIO(ctypes.Structure):
    _fields_ = [(n, _vp) for n in (
        "theta", "C", "c", "X", "U", "dLdX", "dLdU", "dLdJ", "dC", "dc", "dx0", "dtheta",
        "dX", "dU", "fail_t")]


RACE_MAX_GATES = 32


class DiffMPCTrack(ctypes.Structure):
    """include/diffmpc.h DiffMPCTrack (the batched race-environment step)."""
    _fields_ = [
        ("n_gates", ctypes.c_int32), ("laps", ctypes.c_int32), ("dim", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("center", (ctypes.c_double * 3) * RACE_MAX_GATES), ("normal", (ctypes.c_double * 3) * RACE_MAX_GATES),
        ("width", ctypes.c_double * RACE_MAX_GATES), ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
    ] + [(n, ctypes.c_double) for n in ("k_p", "gate_bonus", "crash_penalty", "time_penalty", "progress_cap",
                                         "timeout", "miss_factor", "pos_scale", "vel_scale", "omega_scale")]


def make_track(track, cfg, pos_scale, vel_scale, omega_scale) -> DiffMPCTrack:
    G = len(track.gates)
    if G > RACE_MAX_GATES:
        raise ConfigError(f"at most {RACE_MAX_GATES} gates are supported")
    t = DiffMPCTrack()
    t.n_gates, t.laps, t.dim = G, int(track.laps), int(track.dim)
    for i, g in enumerate(track.gates):
        for a in range(track.dim):
            t.center[i][a] = float(g.center[a])
            t.normal[i][a] = float(g.normal[a])
        t.width[i] = float(g.width)
    for a in range(track.dim):
        t.lo[a], t.hi[a] = float(track.lo[a]), float(track.hi[a])
    for n in ("k_p", "gate_bonus", "crash_penalty", "time_penalty", "progress_cap", "timeout", "miss_factor"):
        setattr(t, n, float(getattr(cfg, n)))
    t.pos_scale, t.vel_scale, t.omega_scale = float(pos_scale), float(vel_scale), float(omega_scale)
    return t


def make_problem(model, settings, B: int, layout: int, theta_stride: int = 0, kernel="auto") -> DiffMPCProblem:
    """Fill a DiffMPCProblem from the reference-style model/settings objects."""
    nu = model.n_u
    if nu > MAX_NU:
        raise ConfigError(f"n_u={nu} exceeds the ABI limit {MAX_NU}")
    if len(settings.alphas) > MAX_ALPHA:
        raise ConfigError(f"at most {MAX_ALPHA} line-search step sizes are supported")
    u_min, u_max = settings.bounds_for(nu)
    p = DiffMPCProblem()
    p.B = int(B)
    p.T = int(settings.T)
    p.nx = int(model.n_x)
    p.nu = int(nu)
    p.model_kind = int(model.kind)
    p.cost_layout = int(layout)
    p.K_max = int(settings.K_max)
    p.n_alpha = len(settings.alphas)
    p.boxqp_max_iter = int(settings.boxqp_max_iter)
    p.n_theta = int(model.params.shape[0])
    p.theta_stride = int(theta_stride)
    p.kernel_select = kernel_code(kernel)
    p.dt = float(model.dt)
    p.conv_tol = float(settings.conv_tol)
    p.boxqp_tol = float(settings.boxqp_tol)
    for i in range(nu):
        p.u_min[i] = float(u_min[i])
        p.u_max[i] = float(u_max[i])
    for i, a in enumerate(settings.alphas):
        p.alphas[i] = float(a)
    return p


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()

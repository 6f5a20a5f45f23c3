"""ctypes front-end of the CPU oracle (oracle/diffmpc_oracle.c).

TEST INFRASTRUCTURE ONLY. Imported exclusively by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg, always as the checker or the
timed CPU baseline — never as part of the product path (which fails loudly when
libdiffmpc.so is missing).

The oracle restates the reference's float64 algorithm (see the C file header for
the file:line map) and is pinned bit-exactly against golden vectors produced by
the unmodified reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2605_29155_b200 import _abi  # noqa: E402  (struct layout only)

LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_forward.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_forward.restype = ctypes.c_int
        L.oracle_backward.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_backward.restype = ctypes.c_int
        L.oracle_dynamics.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 6
        L.oracle_dynamics.restype = ctypes.c_int
        L.oracle_boxqp.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.oracle_boxqp.restype = ctypes.c_int
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def forward(model, settings, x0, C, c, U_warm, layout=_abi.COST_DENSE, threads=1, theta=None):
    """Batch solve; returns a dict of numpy outputs (reference semantics)."""
    x0, C, c, U_warm = _f64(x0), _f64(C), _f64(c), _f64(U_warm)
    B = x0.shape[0]
    T, nx, nu = settings.T, model.n_x, model.n_u
    theta = _f64(model.params if theta is None else theta)
    stride = 0 if theta.ndim == 1 else theta.shape[-1]
    p = _abi.make_problem(model, settings, B, layout, stride)
    out = dict(
        X=np.zeros((B, T + 1, nx)), U=np.zeros((B, T, nu)), J=np.zeros(B),
        K=np.zeros((B, T, nu, nx)), k=np.zeros((B, T, nu)),
        iters=np.zeros(B, np.int32), converged=np.zeros(B, np.uint8),
        diverged=np.zeros(B, np.uint8), fail_t=np.zeros(B, np.int32),
        clamped=np.zeros((B, T, nu), np.uint8), alpha_hist=np.zeros((B, settings.K_max)),
        J_hist=np.zeros((B, settings.K_max + 1)),
    )
    io = _abi.DiffMPCForwardIO()
    for name, arr in (("theta", theta), ("C", C), ("c", c), ("x0", x0), ("U_warm", U_warm)):
        setattr(io, name, arr.ctypes.data)
    for name, arr in out.items():
        setattr(io, name, arr.ctypes.data)
    rc = lib().oracle_forward(ctypes.byref(p), ctypes.byref(io), int(threads))
    if rc != 0:
        raise ValueError("oracle_forward rejected the problem")
    return out


def backward(model, settings, C, c, X, U, dLdX=None, dLdU=None, dLdJ=None,
             layout=_abi.COST_DENSE, threads=1, theta=None, want_theta=True):
    C, c, X, U = _f64(C), _f64(c), _f64(X), _f64(U)
    B = X.shape[0]
    T, nx, nu = settings.T, model.n_x, model.n_u
    nz = nx + nu
    theta = _f64(model.params if theta is None else theta)
    stride = 0 if theta.ndim == 1 else theta.shape[-1]
    p = _abi.make_problem(model, settings, B, layout, stride)
    nth = p.n_theta
    out = dict(
        dC=np.zeros((B, T, nz, nz)) if layout == _abi.COST_DENSE else np.zeros((B, T, nz)),
        dc=np.zeros((B, T, nz)), dx0=np.zeros((B, nx)),
        dX=np.zeros((B, T + 1, nx)), dU=np.zeros((B, T, nu)), fail_t=np.zeros(B, np.int32),
    )
    if want_theta and nth > 0:
        out["dtheta"] = np.zeros((B, nth))
    io = _abi.DiffMPCBackwardIO()
    keep = []
    for name, arr in (("theta", theta), ("C", C), ("c", c), ("X", X), ("U", U),
                      ("dLdX", dLdX), ("dLdU", dLdU), ("dLdJ", dLdJ)):
        if arr is not None:
            arr = _f64(arr)
            keep.append(arr)
            setattr(io, name, arr.ctypes.data)
    for name, arr in out.items():
        setattr(io, name, arr.ctypes.data)
    rc = lib().oracle_backward(ctypes.byref(p), ctypes.byref(io), int(threads))
    if rc != 0:
        raise ValueError("oracle_backward rejected the problem")
    return out


def dynamics(model, x, u, theta=None):
    x, u = _f64(x), _f64(u)
    N = x.shape[0]
    nx, nu = model.n_x, model.n_u
    theta = _f64(model.params if theta is None else theta)
    stride = 0 if theta.ndim == 1 else theta.shape[-1]
    from paper_2605_29155_b200.settings import SolveSettings

    s = SolveSettings(T=1, u_min=-np.ones(nu), u_max=np.ones(nu))
    p = _abi.make_problem(model, s, N, _abi.COST_DENSE, stride)
    xn = np.zeros((N, nx))
    A = np.zeros((N, nx, nx))
    Bm = np.zeros((N, nx, nu))
    lib().oracle_dynamics(ctypes.byref(p), N, theta.ctypes.data, x.ctypes.data, u.ctypes.data,
                          xn.ctypes.data, A.ctypes.data, Bm.ctypes.data)
    return xn, A, Bm


def boxqp(H, g, lo, hi, u0=None, max_iter=100, tol=1e-10):
    """Projected-Newton box QP (kernels.py:239-318); returns (u, free, status)."""
    H, g, lo, hi = _f64(H), _f64(g), _f64(lo), _f64(hi)
    n = g.shape[0]
    u = np.zeros(n) if u0 is None else np.array(u0, dtype=np.float64)
    free = np.zeros(n, np.uint8)
    st = lib().oracle_boxqp(H.ctypes.data, g.ctypes.data, lo.ctypes.data, hi.ctypes.data,
                            u.ctypes.data, free.ctypes.data, n, int(max_iter), float(tol))
    return u, free.astype(bool), st

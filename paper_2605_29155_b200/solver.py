"""Array-level batch API on the GPU (the B200 counterpart of batchexec.solve_raw /
backward_batch_arrays, /root/reference/pkg/src/fusedmpc/batchexec.py:156-186).

Inputs may be numpy arrays or torch tensors (any device); they are moved once to the
CUDA device in the requested dtype, batch-major like the reference workspaces.
Outputs stay on the device as torch tensors. Each call enqueues exactly one kernel on
the current torch CUDA stream (no host synchronisation inside).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi, _lib
from .errors import ConfigError, ExtensionMissingError

_DT = {torch.float32: "f32", torch.float64: "f64"}


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise ExtensionMissingError("no CUDA device: the DiffMPC layer runs only on the GPU")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ConfigError(f"DiffMPC kernels run on CUDA devices, got {device}")
    return device


def _as(t, dtype, device, shape=None, name="array"):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(t))
    elif not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    t = t.to(device=device, dtype=dtype, non_blocking=True).contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ConfigError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


_THETA_CACHE = {}


def _theta(model, theta, dtype, device, B):
    if theta is None:  # the model's own parameters: one device copy per (values, dtype, device)
        key = (np.asarray(model.params, dtype=np.float64).tobytes(), dtype, str(device))
        th = _THETA_CACHE.get(key)
        if th is None:
            th = _THETA_CACHE[key] = _as(model.params, dtype, device)
    else:
        th = _as(theta, dtype, device)
    if th.ndim == 1:
        if th.shape[0] != model.n_theta:
            raise ConfigError(f"theta must have {model.n_theta} entries, got {th.shape[0]}")
        return th, 0
    if th.shape != (B, model.n_theta):
        raise ConfigError(f"per-problem theta must be ({B}, {model.n_theta}), got {tuple(th.shape)}")
    return th, model.n_theta


def _stream(stream=None, device=None) -> int:
    s = torch.cuda.current_stream(device) if stream is None else stream
    return s.cuda_stream


def _on(dev, stream):
    """Run a call with `dev` current and, when given, `stream` as torch's current stream, so
    every allocation of the call (outputs, converted inputs, workspace) is made on the stream
    the kernel runs on and the caching allocator cannot recycle it under the running kernel."""
    import contextlib

    ctx = contextlib.ExitStack()
    ctx.enter_context(torch.cuda.device(dev))
    if stream is not None:
        ctx.enter_context(torch.cuda.stream(stream))
    return ctx


def _layout(C, B, T, nz) -> int:
    if tuple(C.shape) == (B, T, nz, nz):
        return _abi.COST_DENSE
    if tuple(C.shape) == (B, T, nz):
        return _abi.COST_DIAG
    raise ConfigError(f"C must be (B,T,nz,nz) dense or (B,T,nz) diagonal, got {tuple(C.shape)}")


@dataclass
class SolveOutput:
    """Device-resident result of a batched solve (collect_result semantics, ilqr.py:250-268)."""

    X: torch.Tensor           # (B, T+1, nx)
    U: torch.Tensor           # (B, T, nu)
    J: torch.Tensor           # (B,)
    K: torch.Tensor           # (B, T, nu, nx) last computed gains
    k: torch.Tensor           # (B, T, nu)
    iters: torch.Tensor       # (B,) int32
    converged: torch.Tensor   # (B,) bool, converged and not failed
    diverged: torch.Tensor    # (B,) bool
    fail_t: torch.Tensor      # (B,) int32, -1 = ok
    clamped: torch.Tensor     # (B, T, nu) bool, (U<=u_min)|(U>=u_max)
    alpha_hist: torch.Tensor  # (B, K_max)
    J_hist: torch.Tensor      # (B, K_max+1)
    C: torch.Tensor = field(repr=False, default=None)   # the cost tensors used (device)
    c: torch.Tensor = field(repr=False, default=None)
    theta: torch.Tensor = field(repr=False, default=None)
    layout: int = _abi.COST_DENSE

    @property
    def B(self) -> int:
        return self.X.shape[0]

    @property
    def failed(self) -> torch.Tensor:
        return (self.fail_t >= 0) | self.diverged


@dataclass
class GradOutput:
    """Device-resident implicit gradients (GradOutput semantics, gradlayer.py:38-45)."""

    dC: torch.Tensor          # (B,T,nz,nz) dense or (B,T,nz) diagonal
    dc: torch.Tensor          # (B,T,nz)
    dx0: torch.Tensor         # (B,nx)
    dtheta: torch.Tensor | None  # (B,n_theta) per problem
    fail_t: torch.Tensor      # (B,) int32
    dX: torch.Tensor | None = None
    dU: torch.Tensor | None = None


def solve_raw(model, settings, x_init, C, c, U_warm, *, dtype=torch.float32, device=None, theta=None,
              stream=None, want_gains=True, kernel="auto") -> SolveOutput:
    """Batched iLQR solve over stacked cost arrays (batchexec.solve_raw, batchexec.py:156-163).

    C is (B,T,nz,nz) dense or (B,T,nz) diagonal. One kernel launch. ``kernel`` picks the
    forward mapping ("auto" | "throughput" | "latency", see diffmpc.h kernel_select).
    """
    if dtype not in _DT:
        raise ConfigError(f"dtype must be float32 or float64, got {dtype}")
    dev = _device(device)
    with _on(dev, stream):
        return _solve_raw(model, settings, x_init, C, c, U_warm, dtype, dev, theta, want_gains, kernel)


def _solve_raw(model, settings, x_init, C, c, U_warm, dtype, dev, theta, want_gains, kernel):
    T, nx, nu = settings.T, model.n_x, model.n_u
    nz = nx + nu
    x_init = _as(x_init, dtype, dev, name="x_init")
    if x_init.ndim != 2 or x_init.shape[1] != nx:
        raise ConfigError(f"x_init must be (B, {nx}), got {tuple(x_init.shape)}")
    B = x_init.shape[0]
    C = _as(C, dtype, dev, name="C")
    layout = _layout(C, B, T, nz)
    c = _as(c, dtype, dev, (B, T, nz), "c")
    U_warm = _as(U_warm, dtype, dev, (B, T, nu), "U_warm")
    th, stride = _theta(model, theta, dtype, dev, B)
    p = _abi.make_problem(model, settings, B, layout, stride, kernel)
    f = dict(device=dev)
    out = SolveOutput(
        X=torch.empty((B, T + 1, nx), dtype=dtype, **f), U=torch.empty((B, T, nu), dtype=dtype, **f),
        J=torch.empty((B,), dtype=dtype, **f),
        K=torch.empty((B, T, nu, nx), dtype=dtype, **f) if want_gains else None,
        k=torch.empty((B, T, nu), dtype=dtype, **f) if want_gains else None,
        iters=torch.empty((B,), dtype=torch.int32, **f),
        converged=torch.empty((B,), dtype=torch.uint8, **f),
        diverged=torch.empty((B,), dtype=torch.uint8, **f),
        fail_t=torch.empty((B,), dtype=torch.int32, **f),
        clamped=torch.empty((B, T, nu), dtype=torch.uint8, **f),
        alpha_hist=torch.empty((B, settings.K_max), dtype=dtype, **f),
        J_hist=torch.empty((B, settings.K_max + 1), dtype=dtype, **f),
        C=C, c=c, theta=th, layout=layout,
    )
    io = _abi.DiffMPCForwardIO()
    P = _abi.ptr
    io.theta, io.C, io.c, io.x0, io.U_warm = P(th), P(C), P(c), P(x_init), P(U_warm)
    for name in ("X", "U", "J", "K", "k", "iters", "converged", "diverged", "fail_t", "clamped",
                 "alpha_hist", "J_hist"):
        setattr(io, name, P(getattr(out, name)))
    # device workspace (work counter + L2-resident gains) from torch's caching allocator
    L = _lib.lib()
    wsb = int(L.diffmpc_forward_workspace_bytes(ctypes.byref(p), 4 if dtype == torch.float32 else 8))
    ws = torch.empty((wsb,), dtype=torch.uint8, device=dev)
    io.workspace, io.workspace_bytes = P(ws), wsb
    fn = getattr(L, f"diffmpc_forward_{_DT[dtype]}")
    _lib.check(fn(ctypes.byref(p), ctypes.byref(io), _stream()))
    out.converged = out.converged.bool()
    out.diverged = out.diverged.bool()
    out.clamped = out.clamped.bool()
    return out


def solve_diag(model, settings, x_init, diag, cvec, U_warm, **kw) -> SolveOutput:
    """Diagonal cost parameterisation (MpcSolver.solve_diag, policy.py:214-222); the
    diagonal is consumed directly instead of being expanded to dense C."""
    return solve_raw(model, settings, x_init, diag, cvec, U_warm, **kw)


def backward_raw(model, settings, C, c, X, U, dLdX=None, dLdU=None, dLdJ=None, *, dtype=None,
                 device=None, theta=None, want_theta=False, want_traj=False, stream=None) -> GradOutput:
    """Implicit backward through a solution (relinearisation + aux LQR + assembly,
    policy.py:252-283 / gradlayer.py:98-150), plus dtheta / dL/dJ terms. One launch."""
    dev = _device(device)
    if dtype is None:
        dtype = X.dtype if isinstance(X, torch.Tensor) else torch.float32
    with _on(dev, stream):
        return _backward_raw(model, settings, C, c, X, U, dLdX, dLdU, dLdJ, dtype, dev, theta, want_theta,
                             want_traj)


def _backward_raw(model, settings, C, c, X, U, dLdX, dLdU, dLdJ, dtype, dev, theta, want_theta, want_traj):
    T, nx, nu = settings.T, model.n_x, model.n_u
    nz = nx + nu
    X = _as(X, dtype, dev, name="X")
    B = X.shape[0]
    if tuple(X.shape) != (B, T + 1, nx):
        raise ConfigError(f"X must be ({B}, {T + 1}, {nx}), got {tuple(X.shape)}")
    U = _as(U, dtype, dev, (B, T, nu), "U")
    C = _as(C, dtype, dev, name="C")
    layout = _layout(C, B, T, nz)
    c = _as(c, dtype, dev, (B, T, nz), "c") if c is not None else None
    dLdX = _as(dLdX, dtype, dev, (B, T + 1, nx), "dL/dX")
    dLdU = _as(dLdU, dtype, dev, (B, T, nu), "dL/dU")
    dLdJ = _as(dLdJ, dtype, dev, (B,), "dL/dJ")
    th, stride = _theta(model, theta, dtype, dev, B)
    if (want_theta or dLdJ is not None) and c is None:
        raise ConfigError("c is required for dtheta / dL/dJ gradients")
    p = _abi.make_problem(model, settings, B, layout, stride)
    f = dict(device=dev, dtype=dtype)
    out = GradOutput(
        dC=torch.empty(tuple(C.shape), **f), dc=torch.empty((B, T, nz), **f),
        dx0=torch.empty((B, nx), **f),
        dtheta=torch.empty((B, model.n_theta), **f) if (want_theta and model.n_theta > 0) else None,
        fail_t=torch.empty((B,), device=dev, dtype=torch.int32),
        dX=torch.empty((B, T + 1, nx), **f) if want_traj else None,
        dU=torch.empty((B, T, nu), **f) if want_traj else None,
    )
    io = _abi.DiffMPCBackwardIO()
    P = _abi.ptr
    io.theta, io.C, io.c, io.X, io.U = P(th), P(C), P(c), P(X), P(U)
    io.dLdX, io.dLdU, io.dLdJ = P(dLdX), P(dLdU), P(dLdJ)
    io.dC, io.dc, io.dx0, io.dtheta = P(out.dC), P(out.dc), P(out.dx0), P(out.dtheta)
    io.dX, io.dU, io.fail_t = P(out.dX), P(out.dU), P(out.fail_t)
    fn = getattr(_lib.lib(), f"diffmpc_backward_{_DT[dtype]}")
    _lib.check(fn(ctypes.byref(p), ctypes.byref(io), _stream()))
    return out


def to_numpy(t):
    """Device tensor -> numpy through page-locked memory (torch's caching host allocator):
    one DMA at PCIe rate instead of a pageable copy (≈ 2-6 GB/s for the 0.1-0.2 GB dC of a
    16k batch). The array views the pinned buffer, which returns to the cache when freed."""
    if t is None:
        return None
    if not t.is_cuda:
        return t.numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def dynamics(model, x, u, *, dtype=torch.float64, device=None, want_jac=True, theta=None):
    """Batched f(x,u) and Jacobians on the GPU; returns numpy arrays (N,nx), (N,nx,nx), (N,nx,nu)."""
    return tuple(to_numpy(t) for t in dynamics_t(model, x, u, dtype=dtype, device=device, want_jac=want_jac,
                                           theta=theta))


def dynamics_t(model, x, u, *, dtype=torch.float64, device=None, want_jac=False, theta=None):
    """Device-resident variant of ``dynamics``: returns torch tensors (xn, A, Bm) on the device,
    enqueued on the current stream (used by the batched environment step)."""
    dev = _device(device)
    nx, nu = model.n_x, model.n_u
    x = _as(x, dtype, dev, name="x")
    N = x.shape[0]
    u = _as(u, dtype, dev, (N, nu), "u")
    th, stride = _theta(model, theta, dtype, dev, N)
    from .settings import SolveSettings

    s = SolveSettings(T=1, u_min=-np.ones(nu), u_max=np.ones(nu))
    p = _abi.make_problem(model, s, N, _abi.COST_DENSE, stride)
    xn = torch.empty((N, nx), device=dev, dtype=dtype)
    A = torch.empty((N, nx, nx), device=dev, dtype=dtype) if want_jac else None
    Bm = torch.empty((N, nx, nu), device=dev, dtype=dtype) if want_jac else None
    fn = getattr(_lib.lib(), f"diffmpc_dynamics_{_DT[dtype]}")
    P = _abi.ptr
    with torch.cuda.device(dev):
        _lib.check(fn(ctypes.byref(p), N, P(th), P(x), P(u), P(xn), P(A), P(Bm), _stream()))
    return xn, A, Bm


class SolvePlan:
    """Preallocated forward (and backward) launches for a fixed problem shape.

    ``solve_raw`` allocates its outputs and builds the ABI structs on every call (~0.1 ms of
    host time — as much as a B=1 solve on the GPU). A plan does that once: outputs, gradient
    buffers and the workspace are allocated up front, the ``DiffMPCProblem`` / IO structs are
    filled once, and each call only patches the input pointers and enqueues the kernel(s).
    Inputs must be contiguous device tensors of the plan's dtype and shapes; the returned
    SolveOutput / GradOutput are the plan's own buffers (overwritten by the next call).
    """

    def __init__(self, model, settings, B, *, layout="dense", dtype=torch.float32, device=None, theta=None,
                 want_gains=True, backward=True, kernel="auto"):
        if dtype not in _DT:
            raise ConfigError(f"dtype must be float32 or float64, got {dtype}")
        self.dev = _device(device)
        if self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        self.model, self.settings, self.B, self.dtype = model, settings, int(B), dtype
        T, nx, nu = settings.T, model.n_x, model.n_u
        nz = nx + nu
        self.layout = _abi.COST_DENSE if layout == "dense" else _abi.COST_DIAG
        self.C_shape = (self.B, T, nz, nz) if self.layout == _abi.COST_DENSE else (self.B, T, nz)
        self.theta, stride = _theta(model, theta, dtype, self.dev, self.B)
        self.p = _abi.make_problem(model, settings, self.B, self.layout, stride, kernel)
        f = dict(device=self.dev)
        self.out = SolveOutput(
            X=torch.empty((B, T + 1, nx), dtype=dtype, **f), U=torch.empty((B, T, nu), dtype=dtype, **f),
            J=torch.empty((B,), dtype=dtype, **f),
            K=torch.empty((B, T, nu, nx), dtype=dtype, **f) if want_gains else None,
            k=torch.empty((B, T, nu), dtype=dtype, **f) if want_gains else None,
            iters=torch.empty((B,), dtype=torch.int32, **f), converged=torch.empty((B,), dtype=torch.uint8, **f),
            diverged=torch.empty((B,), dtype=torch.uint8, **f), fail_t=torch.empty((B,), dtype=torch.int32, **f),
            clamped=torch.empty((B, T, nu), dtype=torch.uint8, **f),
            alpha_hist=torch.empty((B, settings.K_max), dtype=dtype, **f),
            J_hist=torch.empty((B, settings.K_max + 1), dtype=dtype, **f), theta=self.theta, layout=self.layout)
        L = _lib.lib()
        P = _abi.ptr
        wsb = int(L.diffmpc_forward_workspace_bytes(ctypes.byref(self.p), 4 if dtype == torch.float32 else 8))
        self.ws = torch.empty((wsb,), dtype=torch.uint8, **f)
        self.fio = _abi.DiffMPCForwardIO()
        self.fio.theta = P(self.theta)
        for name in ("X", "U", "J", "K", "k", "iters", "converged", "diverged", "fail_t", "clamped",
                     "alpha_hist", "J_hist"):
            setattr(self.fio, name, P(getattr(self.out, name)))
        self.fio.workspace, self.fio.workspace_bytes = P(self.ws), wsb
        self._fwd = getattr(L, f"diffmpc_forward_{_DT[dtype]}")
        self.grad = None
        if backward:
            self.grad = GradOutput(dC=torch.empty(self.C_shape, dtype=dtype, **f),
                                   dc=torch.empty((B, T, nz), dtype=dtype, **f),
                                   dx0=torch.empty((B, nx), dtype=dtype, **f), dtheta=None,
                                   fail_t=torch.empty((B,), dtype=torch.int32, **f))
            self.bio = _abi.DiffMPCBackwardIO()
            self.bio.theta = P(self.theta)
            self.bio.dC, self.bio.dc, self.bio.dx0 = P(self.grad.dC), P(self.grad.dc), P(self.grad.dx0)
            self.bio.fail_t = P(self.grad.fail_t)
            self._bwd = getattr(L, f"diffmpc_backward_{_DT[dtype]}")

    def _check(self, t, shape, name):
        if (not isinstance(t, torch.Tensor) or t.dtype != self.dtype or t.device != self.dev
                or tuple(t.shape) != tuple(shape) or not t.is_contiguous()):
            raise ConfigError(f"{name}: expected a contiguous {self.dtype} tensor of shape {tuple(shape)} on {self.dev}")
        return t.data_ptr()

    def solve(self, x_init, C, c, U_warm, stream=None) -> SolveOutput:
        T, nx, nu = self.settings.T, self.model.n_x, self.model.n_u
        io = self.fio
        io.x0 = self._check(x_init, (self.B, nx), "x_init")
        io.C = self._check(C, self.C_shape, "C")
        io.c = self._check(c, (self.B, T, nx + nu), "c")
        io.U_warm = self._check(U_warm, (self.B, T, nu), "U_warm")
        # the plan's buffers are owned by the plan (no per-call allocation); the launch goes
        # to `stream` or the current stream of the PLAN's device
        _lib.check(self._fwd(ctypes.byref(self.p), ctypes.byref(io), _stream(stream, self.dev)))
        self.out.C, self.out.c = C, c
        return self.out

    def backward(self, dLdX=None, dLdU=None, dLdJ=None, stream=None) -> GradOutput:
        """Implicit backward at the last ``solve`` of this plan (its C, c, X, U)."""
        if self.grad is None:
            raise ConfigError("plan was built with backward=False")
        T, nx, nu = self.settings.T, self.model.n_x, self.model.n_u
        io, o = self.bio, self.out
        io.C, io.c, io.X, io.U = o.C.data_ptr(), o.c.data_ptr(), o.X.data_ptr(), o.U.data_ptr()
        io.dLdX = None if dLdX is None else self._check(dLdX, (self.B, T + 1, nx), "dL/dX")
        io.dLdU = None if dLdU is None else self._check(dLdU, (self.B, T, nu), "dL/dU")
        io.dLdJ = None if dLdJ is None else self._check(dLdJ, (self.B,), "dL/dJ")
        _lib.check(self._bwd(ctypes.byref(self.p), ctypes.byref(io), _stream(stream, self.dev)))
        return self.grad

"""Model plug-in that lets the UNMODIFIED reference orchestrator solve the 13-state
quadrotor (golden-vector generation only; runs in the build container where
/root/reference is importable).

The reference has no 13-state model. Its orchestrator
(ilqr.run_staged_solve, ilqr.py:154-247) and the layer backward
(policy.MpcSolveLayer.backward, policy.py:252-283) resolve the three model-bound
range kernels as ``kernels.<name>`` at call time, so swapping those three
attributes routes the quadrotor through the reference's own Riccati/boxQP/
line-search/aux code (probe P3).

The restated range kernels keep the reference's control flow exactly
(kernels.py:161-187 rollout/linearize, 520-574 line search: cost before step,
clamp order ``v<lo ... elif v>hi``, the dead rule); only the model calls change.
The model expression trees are token-for-token the ones in
oracle/diffmpc_oracle.c (quad13_step / quad13_jac), so the C oracle can be pinned
bit-exactly against these goldens.
"""

import math

import numpy as np
from numba import njit

from fusedmpc import kernels as K

KIND_QUAD13 = 3
INV_SQRT2 = 0.7071067811865476
_J = dict(cache=False, nogil=True)


@njit(**_J)
def quad13_step(mp, dt, x, u, out):
    m = mp[0]; l = mp[1]; Jx = mp[2]; Jy = mp[3]; Jz = mp[4]; kap = mp[5]; g = mp[6]
    d = l * INV_SQRT2
    qw = x[3]; qx = x[4]; qy = x[5]; qz = x[6]
    wx = x[10]; wy = x[11]; wz = x[12]
    F = ((u[0] + u[1]) + u[2]) + u[3]
    tx = d * (((u[0] + u[1]) - u[2]) - u[3])
    ty = d * (((u[1] - u[0]) + u[2]) - u[3])
    tz = kap * (((u[0] - u[1]) + u[2]) - u[3])
    hw = 0.5 * dt
    r13 = 2.0 * (qx * qz + qw * qy)
    r23 = 2.0 * (qy * qz - qw * qx)
    r33 = 1.0 - 2.0 * (qx * qx + qy * qy)
    a = F / m
    out[0] = x[0] + dt * x[7]
    out[1] = x[1] + dt * x[8]
    out[2] = x[2] + dt * x[9]
    out[3] = qw + hw * (((-qx * wx) - qy * wy) - qz * wz)
    out[4] = qx + hw * ((qw * wx + qy * wz) - qz * wy)
    out[5] = qy + hw * ((qw * wy - qx * wz) + qz * wx)
    out[6] = qz + hw * ((qw * wz + qx * wy) - qy * wx)
    out[7] = x[7] + dt * (r13 * a)
    out[8] = x[8] + dt * (r23 * a)
    out[9] = x[9] + dt * (r33 * a - g)
    out[10] = wx + dt * ((tx - (Jz - Jy) * wy * wz) / Jx)
    out[11] = wy + dt * ((ty - (Jx - Jz) * wz * wx) / Jy)
    out[12] = wz + dt * ((tz - (Jy - Jx) * wx * wy) / Jz)


@njit(**_J)
def quad13_jac(mp, dt, x, u, A, B):
    m = mp[0]; l = mp[1]; Jx = mp[2]; Jy = mp[3]; Jz = mp[4]; kap = mp[5]
    d = l * INV_SQRT2
    qw = x[3]; qx = x[4]; qy = x[5]; qz = x[6]
    wx = x[10]; wy = x[11]; wz = x[12]
    F = ((u[0] + u[1]) + u[2]) + u[3]
    hw = 0.5 * dt
    a = F / m
    r13 = 2.0 * (qx * qz + qw * qy)
    r23 = 2.0 * (qy * qz - qw * qx)
    r33 = 1.0 - 2.0 * (qx * qx + qy * qy)
    for i in range(13):
        for j in range(13):
            A[i, j] = 0.0
        for j in range(4):
            B[i, j] = 0.0
        A[i, i] = 1.0
    A[0, 7] = dt; A[1, 8] = dt; A[2, 9] = dt
    A[3, 4] = -hw * wx; A[3, 5] = -hw * wy; A[3, 6] = -hw * wz
    A[3, 10] = -hw * qx; A[3, 11] = -hw * qy; A[3, 12] = -hw * qz
    A[4, 3] = hw * wx; A[4, 5] = hw * wz; A[4, 6] = -hw * wy
    A[4, 10] = hw * qw; A[4, 11] = -hw * qz; A[4, 12] = hw * qy
    A[5, 3] = hw * wy; A[5, 4] = -hw * wz; A[5, 6] = hw * wx
    A[5, 10] = hw * qz; A[5, 11] = hw * qw; A[5, 12] = -hw * qx
    A[6, 3] = hw * wz; A[6, 4] = hw * wy; A[6, 5] = -hw * wx
    A[6, 10] = -hw * qy; A[6, 11] = hw * qx; A[6, 12] = hw * qw
    da = dt * a
    A[7, 3] = da * (2.0 * qy); A[7, 4] = da * (2.0 * qz)
    A[7, 5] = da * (2.0 * qw); A[7, 6] = da * (2.0 * qx)
    A[8, 3] = da * (-2.0 * qx); A[8, 4] = da * (-2.0 * qw)
    A[8, 5] = da * (2.0 * qz); A[8, 6] = da * (2.0 * qy)
    A[9, 4] = da * (-4.0 * qx); A[9, 5] = da * (-4.0 * qy)
    b7 = dt * r13 / m
    b8 = dt * r23 / m
    b9 = dt * r33 / m
    for j in range(4):
        B[7, j] = b7
        B[8, j] = b8
        B[9, j] = b9
    A[10, 11] = -dt * ((Jz - Jy) * wz) / Jx; A[10, 12] = -dt * ((Jz - Jy) * wy) / Jx
    A[11, 10] = -dt * ((Jx - Jz) * wz) / Jy; A[11, 12] = -dt * ((Jx - Jz) * wx) / Jy
    A[12, 10] = -dt * ((Jy - Jx) * wy) / Jz; A[12, 11] = -dt * ((Jy - Jx) * wx) / Jz
    bx = dt * d / Jx
    by = dt * d / Jy
    bz = dt * kap / Jz
    B[10, 0] = bx; B[10, 1] = bx; B[10, 2] = -bx; B[10, 3] = -bx
    B[11, 0] = -by; B[11, 1] = by; B[11, 2] = by; B[11, 3] = -by
    B[12, 0] = bz; B[12, 1] = -bz; B[12, 2] = bz; B[12, 3] = -bz


@njit(**_J)
def _step(kind, mp, dt, x, u, out):
    if kind == KIND_QUAD13:
        quad13_step(mp, dt, x, u, out)
    else:
        K.step_one(kind, mp, dt, x, u, out)


@njit(**_J)
def _jac(kind, mp, dt, x, u, A, B):
    if kind == KIND_QUAD13:
        quad13_jac(mp, dt, x, u, A, B)
    else:
        K.jac_one(kind, mp, dt, x, u, A, B)


@njit(**_J)
def rollout_range(kind, mp, dt, X, U, C, c, J, fail_t, active, i_lo, i_hi, t_lo, t_hi):
    for i in range(i_lo, i_hi):
        if active[i] == 0:
            continue
        for t in range(t_lo, t_hi):
            J[i] += K._stage_cost_xu(C[i, t], c[i, t], X[i, t], U[i, t])
            _step(kind, mp, dt, X[i, t], U[i, t], X[i, t + 1])
            if not K._finite_vec(X[i, t + 1]):
                fail_t[i] = t
                active[i] = 0
                J[i] = np.inf
                break


@njit(**_J)
def linearize_range(kind, mp, dt, X, U, A, B, active, i_lo, i_hi, t_lo, t_hi):
    for i in range(i_lo, i_hi):
        if active[i] != 0:
            for t in range(t_lo, t_hi):
                _jac(kind, mp, dt, X[i, t], U[i, t], A[i, t], B[i, t])


@njit(**_J)
def linesearch_range(kind, mp, dt, Xnom, Unom, Kg, kg, alphas, u_min, u_max, C, c,
                     Xc, Uc, Jc, dead, active, c_lo, c_hi, t_lo, t_hi):
    n_alpha = alphas.shape[0]
    n_u = Unom.shape[2]
    n_x = Xnom.shape[2]
    for ci in range(c_lo, c_hi):
        i = ci // n_alpha
        a = ci % n_alpha
        if active[i] == 0 or dead[i, a] == 1:
            continue
        alpha = alphas[a]
        for t in range(t_lo, t_hi):
            xc = Xc[i, a, t]
            for r in range(n_u):
                v = Unom[i, t, r] + alpha * kg[i, t, r]
                for b in range(n_x):
                    v += Kg[i, t, r, b] * (xc[b] - Xnom[i, t, b])
                if v < u_min[r]:
                    v = u_min[r]
                elif v > u_max[r]:
                    v = u_max[r]
                Uc[i, a, t, r] = v
            Jc[i, a] += K._stage_cost_xu(C[i, t], c[i, t], xc, Uc[i, a, t])
            _step(kind, mp, dt, xc, Uc[i, a, t], Xc[i, a, t + 1])
            if not K._finite_vec(Xc[i, a, t + 1]) or not math.isfinite(Jc[i, a]):
                dead[i, a] = 1
                Jc[i, a] = np.inf
                break


def install():
    """Route the reference's three model-bound range kernels through the plug-in."""
    K.rollout_range = rollout_range
    K.linearize_range = linearize_range
    K.linesearch_range = linesearch_range

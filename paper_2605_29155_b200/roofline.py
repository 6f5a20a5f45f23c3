"""Canonical algorithmic FLOP / byte model of the DiffMPC layer.

Per stage (n = n_x, m = n_u, n_z = n + m; 1 FMA = 2 flop; dense C):
    F_cost = 2 n_z^2 + 3 n_z
    F_ric  = 2n_z^2 + 2n^2 + 2nm + 2n^3 + 2n^2 m + 2n^3 + 2n^2 m + 2nm^2 + m^3/3
             + 2m^2(n+1) + 2m^2 + 4nm + 2m^2 n + 4n^2 m + 3n^2
    F_ls   = 2nm + 2m + F_cost                      (per line-search candidate)
    F_aux  = (F_ric - 2n_z^2) + (4nm + 2n^2) + (3n_z^2 + n_z)
Per solve: fwd = T F_cost + K_it T (F_ric + n_alpha F_ls);  bwd = T F_aux.
Excluded (lower bound): box-QP inner iterations, lambda retries, model f / Jacobians.
Bytes (4 B per element in f32): fwd reads C, c, x0, U_warm and writes X, U, J; bwd reads
dL/dX, dL/dU, C, X, U and writes dC, dc, dx0. The diagonal layout replaces T n_z^2 by
T n_z for C and dC.
"""

from __future__ import annotations

import numpy as np


def stage_flops(n: int, m: int):
    nz = n + m
    F_cost = 2 * nz * nz + 3 * nz
    F_ric = (2 * nz * nz + 2 * n * n + 2 * n * m + 2 * n ** 3 + 2 * n * n * m + 2 * n ** 3
             + 2 * n * n * m + 2 * n * m * m + m ** 3 / 3 + 2 * m * m * (n + 1) + 2 * m * m
             + 4 * n * m + 2 * m * m * n + 4 * n * n * m + 3 * n * n)
    F_ls = 2 * n * m + 2 * m + F_cost
    F_aux = (F_ric - 2 * nz * nz) + (4 * n * m + 2 * n * n) + (3 * nz * nz + nz)
    return F_cost, F_ric, F_ls, F_aux


def fwd_flops(n, m, T, iters, n_alpha=4) -> float:
    """Total forward flops for a batch with per-instance iteration counts `iters`."""
    F_cost, F_ric, F_ls, _ = stage_flops(n, m)
    iters = np.asarray(iters, dtype=np.float64)
    return float(np.sum(T * F_cost + iters * T * (F_ric + n_alpha * F_ls)))


def bwd_flops(n, m, T, B) -> float:
    return float(B * T * stage_flops(n, m)[3])


def fwd_bytes(n, m, T, B, diag=False, elem=4) -> float:
    nz = n + m
    C = T * (nz if diag else nz * nz)
    per = C + T * nz + n + T * m + (T + 1) * n + T * m + 1
    return float(B * per * elem)


def bwd_bytes(n, m, T, B, diag=False, elem=4) -> float:
    nz = n + m
    C = T * (nz if diag else nz * nz)
    per = (T + 1) * n + T * m + C + (T + 1) * n + T * m + C + T * nz + n
    return float(B * per * elem)

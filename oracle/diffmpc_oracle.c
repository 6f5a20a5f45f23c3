/*
 * diffmpc_oracle.c — CPU ORACLE (test infrastructure only; never the product path).
 *
 * A float64 restatement, in plain C, of the reference's DiffMPC hot path
 * (/root/reference/pkg/src/fusedmpc). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and only
 * as the checker or the timed CPU baseline.
 *
 * Parity pin: tests/golden/make_golden.py runs the unmodified reference (imported
 * from /root/reference in the build container) and commits its outputs; the
 * CPU test suite checks this oracle against them BIT-EXACTLY for the reference's
 * own models (compile with -ffp-contract=off so no FMA contraction changes the
 * rounding; numba does not contract either). The 13-state quadrotor has no
 * reference model: its goldens come from the reference orchestrator with the
 * model plugged in by monkeypatch. The dynamics-parameter and
 * optimal-cost gradients are a reference NON-GOAL: parity for those
 * is UNPINNED by the reference and is instead pinned by finite differences on
 * linear models in the tests.
 *
 * Per-instance semantics follow the batch loop exactly: the reference's batch
 * iteration (ilqr.py:204-244) only ever touches an instance while it is active,
 * and inactive instances never reactivate, so running each instance's loop to
 * completion independently yields identical numbers (the reference's own
 * batch==single test, tests/test_batchexec.py:55-62).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/diffmpc.h"

#define MAXN 32 /* max nx + nu handled by the oracle */

static const double ARMIJO = 0.1;    /* kernels.py:31 */
static const double STEP_DEC = 0.6;  /* kernels.py:32 */
static const double MIN_STEP = 1e-20;/* kernels.py:33 */
static const double LAM_INIT = 1e-6; /* kernels.py:34 */
static const double LAM_MAX = 1e-2;  /* kernels.py:35 */
static const double INV_SQRT2 = 0.7071067811865476;

/* ------------------------------------------------------------------------- */
/* dynamics: kernels.py:43-117 (kinds 0-2) and the 13-state quadrotor (kind 3) */
/* ------------------------------------------------------------------------- */

typedef struct {
  int kind, nx, nu;
  double dt;
  const double* mp;
} Model;

/* quadrotor-13: x = [p(3), q(4: w,x,y,z), v(3), w_body(3)], u = 4 rotor thrusts,
 * theta = [m, arm, Jx, Jy, Jz, kappa, g]; X-configuration mixer. Explicit Euler.
 * The expression trees here are mirrored token-for-token by the numba plug-in in
 * tests/golden/quad13_plugin.py and the CUDA model in csrc/models.cuh. */
static void quad13_step(const double* mp, double dt, const double* x, const double* u, double* out) {
  double m = mp[0], l = mp[1], Jx = mp[2], Jy = mp[3], Jz = mp[4], kap = mp[5], g = mp[6];
  double d = l * INV_SQRT2;
  double qw = x[3], qx = x[4], qy = x[5], qz = x[6];
  double wx = x[10], wy = x[11], wz = x[12];
  double F = ((u[0] + u[1]) + u[2]) + u[3];
  double tx = d * (((u[0] + u[1]) - u[2]) - u[3]);
  double ty = d * (((u[1] - u[0]) + u[2]) - u[3]);
  double tz = kap * (((u[0] - u[1]) + u[2]) - u[3]);
  double hw = 0.5 * dt;
  double r13 = 2.0 * (qx * qz + qw * qy);
  double r23 = 2.0 * (qy * qz - qw * qx);
  double r33 = 1.0 - 2.0 * (qx * qx + qy * qy);
  double a = F / m;
  out[0] = x[0] + dt * x[7];
  out[1] = x[1] + dt * x[8];
  out[2] = x[2] + dt * x[9];
  out[3] = qw + hw * (((-qx * wx) - qy * wy) - qz * wz);
  out[4] = qx + hw * ((qw * wx + qy * wz) - qz * wy);
  out[5] = qy + hw * ((qw * wy - qx * wz) + qz * wx);
  out[6] = qz + hw * ((qw * wz + qx * wy) - qy * wx);
  out[7] = x[7] + dt * (r13 * a);
  out[8] = x[8] + dt * (r23 * a);
  out[9] = x[9] + dt * (r33 * a - g);
  out[10] = wx + dt * ((tx - (Jz - Jy) * wy * wz) / Jx);
  out[11] = wy + dt * ((ty - (Jx - Jz) * wz * wx) / Jy);
  out[12] = wz + dt * ((tz - (Jy - Jx) * wx * wy) / Jz);
}

static void quad13_jac(const double* mp, double dt, const double* x, const double* u, double* A, double* B) {
  const int n = 13;
  double m = mp[0], l = mp[1], Jx = mp[2], Jy = mp[3], Jz = mp[4], kap = mp[5];
  double d = l * INV_SQRT2;
  double qw = x[3], qx = x[4], qy = x[5], qz = x[6];
  double wx = x[10], wy = x[11], wz = x[12];
  double F = ((u[0] + u[1]) + u[2]) + u[3];
  double hw = 0.5 * dt;
  double a = F / m;
  double r13 = 2.0 * (qx * qz + qw * qy);
  double r23 = 2.0 * (qy * qz - qw * qx);
  double r33 = 1.0 - 2.0 * (qx * qx + qy * qy);
  for (int i = 0; i < n * n; i++) A[i] = 0.0;
  for (int i = 0; i < n * 4; i++) B[i] = 0.0;
  for (int i = 0; i < n; i++) A[i * n + i] = 1.0;
  A[0 * n + 7] = dt; A[1 * n + 8] = dt; A[2 * n + 9] = dt;
  /* quaternion kinematics rows 3..6 */
  A[3 * n + 4] = -hw * wx; A[3 * n + 5] = -hw * wy; A[3 * n + 6] = -hw * wz;
  A[3 * n + 10] = -hw * qx; A[3 * n + 11] = -hw * qy; A[3 * n + 12] = -hw * qz;
  A[4 * n + 3] = hw * wx; A[4 * n + 5] = hw * wz; A[4 * n + 6] = -hw * wy;
  A[4 * n + 10] = hw * qw; A[4 * n + 11] = -hw * qz; A[4 * n + 12] = hw * qy;
  A[5 * n + 3] = hw * wy; A[5 * n + 4] = -hw * wz; A[5 * n + 6] = hw * wx;
  A[5 * n + 10] = hw * qz; A[5 * n + 11] = hw * qw; A[5 * n + 12] = -hw * qx;
  A[6 * n + 3] = hw * wz; A[6 * n + 4] = hw * wy; A[6 * n + 5] = -hw * wx;
  A[6 * n + 10] = -hw * qy; A[6 * n + 11] = hw * qx; A[6 * n + 12] = hw * qw;
  /* translational rows 7..9: v += dt * R(q) e3 * F/m */
  double da = dt * a;
  A[7 * n + 3] = da * (2.0 * qy); A[7 * n + 4] = da * (2.0 * qz);
  A[7 * n + 5] = da * (2.0 * qw); A[7 * n + 6] = da * (2.0 * qx);
  A[8 * n + 3] = da * (-2.0 * qx); A[8 * n + 4] = da * (-2.0 * qw);
  A[8 * n + 5] = da * (2.0 * qz); A[8 * n + 6] = da * (2.0 * qy);
  A[9 * n + 4] = da * (-4.0 * qx); A[9 * n + 5] = da * (-4.0 * qy);
  double b7 = dt * r13 / m, b8 = dt * r23 / m, b9 = dt * r33 / m;
  for (int j = 0; j < 4; j++) { B[7 * 4 + j] = b7; B[8 * 4 + j] = b8; B[9 * 4 + j] = b9; }
  /* rotational rows 10..12 */
  A[10 * n + 11] = -dt * ((Jz - Jy) * wz) / Jx; A[10 * n + 12] = -dt * ((Jz - Jy) * wy) / Jx;
  A[11 * n + 10] = -dt * ((Jx - Jz) * wz) / Jy; A[11 * n + 12] = -dt * ((Jx - Jz) * wx) / Jy;
  A[12 * n + 10] = -dt * ((Jy - Jx) * wy) / Jz; A[12 * n + 11] = -dt * ((Jy - Jx) * wx) / Jz;
  double bx = dt * d / Jx, by = dt * d / Jy, bz = dt * kap / Jz;
  B[10 * 4 + 0] = bx; B[10 * 4 + 1] = bx; B[10 * 4 + 2] = -bx; B[10 * 4 + 3] = -bx;
  B[11 * 4 + 0] = -by; B[11 * 4 + 1] = by; B[11 * 4 + 2] = by; B[11 * 4 + 3] = -by;
  B[12 * 4 + 0] = bz; B[12 * 4 + 1] = -bz; B[12 * 4 + 2] = bz; B[12 * 4 + 3] = -bz;
}

/* kernels.py:43-73 */
static void step_one(const Model* md, const double* x, const double* u, double* out) {
  int nx = md->nx, nu = md->nu;
  double dt = md->dt;
  const double* mp = md->mp;
  if (md->kind == DIFFMPC_KIND_DOUBLE_INTEGRATOR) {
    int d = nu;
    for (int i = 0; i < d; i++) {
      out[i] = x[i] + dt * x[d + i];
      out[d + i] = x[d + i] + dt * u[i];
    }
  } else if (md->kind == DIFFMPC_KIND_PLANAR_QUADROTOR) {
    double m = mp[0], arm = mp[1], inertia = mp[2], g = mp[3];
    double s = sin(x[2]), c = cos(x[2]);
    double thrust = u[0] + u[1];
    out[0] = x[0] + dt * x[3];
    out[1] = x[1] + dt * x[4];
    out[2] = x[2] + dt * x[5];
    out[3] = x[3] + dt * (-thrust * s / m);
    out[4] = x[4] + dt * (thrust * c / m - g);
    out[5] = x[5] + dt * (arm * (u[1] - u[0]) / inertia);
  } else if (md->kind == DIFFMPC_KIND_LINEAR) {
    for (int i = 0; i < nx; i++) {
      double acc = 0.0;
      for (int j = 0; j < nx; j++) acc += mp[i * nx + j] * x[j];
      for (int j = 0; j < nu; j++) acc += mp[nx * nx + i * nu + j] * u[j];
      out[i] = acc;
    }
  } else {
    quad13_step(mp, dt, x, u, out);
  }
}

/* kernels.py:76-117; A (nx,nx), B (nx,nu) row-major */
static void jac_one(const Model* md, const double* x, const double* u, double* A, double* B) {
  int nx = md->nx, nu = md->nu;
  double dt = md->dt;
  const double* mp = md->mp;
  if (md->kind == DIFFMPC_KIND_QUADROTOR13) { quad13_jac(mp, dt, x, u, A, B); return; }
  for (int i = 0; i < nx; i++) {
    for (int j = 0; j < nx; j++) A[i * nx + j] = 0.0;
    for (int j = 0; j < nu; j++) B[i * nu + j] = 0.0;
  }
  if (md->kind == DIFFMPC_KIND_DOUBLE_INTEGRATOR) {
    int d = nu;
    for (int i = 0; i < nx; i++) A[i * nx + i] = 1.0;
    for (int i = 0; i < d; i++) {
      A[i * nx + d + i] = dt;
      B[(d + i) * nu + i] = dt;
    }
  } else if (md->kind == DIFFMPC_KIND_PLANAR_QUADROTOR) {
    double m = mp[0], arm = mp[1], inertia = mp[2];
    double s = sin(x[2]), c = cos(x[2]);
    double thrust = u[0] + u[1];
    for (int i = 0; i < 6; i++) A[i * 6 + i] = 1.0;
    A[0 * 6 + 3] = dt; A[1 * 6 + 4] = dt; A[2 * 6 + 5] = dt;
    A[3 * 6 + 2] = -dt * thrust * c / m;
    A[4 * 6 + 2] = -dt * thrust * s / m;
    B[3 * 2 + 0] = -dt * s / m; B[3 * 2 + 1] = -dt * s / m;
    B[4 * 2 + 0] = dt * c / m;  B[4 * 2 + 1] = dt * c / m;
    B[5 * 2 + 0] = -dt * arm / inertia; B[5 * 2 + 1] = dt * arm / inertia;
  } else {
    for (int i = 0; i < nx; i++) {
      for (int j = 0; j < nx; j++) A[i * nx + j] = mp[i * nx + j];
      for (int j = 0; j < nu; j++) B[i * nu + j] = mp[nx * nx + i * nu + j];
    }
  }
}

/* ---------------------------------------------------------------------------
 * dtheta contributions (NEW): for one stage,
 *   g_p += lh_i * df_i/dtheta_p  +  lam_i * sum_j d2f_i/(dtheta_p dz_j) dz_j
 * with lh = lambda_hat_{t+1}, lam = lambda_{t+1}. Linear kind: theta = [A, B]
 * entries, df_i/dA_ij = x_j, d(A dz)_i/dA_ij = dx_j (and likewise for B).
 * ------------------------------------------------------------------------- */
static void theta_grad_stage(const Model* md, const double* x, const double* u, const double* dx,
                             const double* du, const double* lh, const double* lam, double* g) {
  int nx = md->nx, nu = md->nu;
  double dt = md->dt;
  const double* mp = md->mp;
  if (md->kind == DIFFMPC_KIND_LINEAR) {
    for (int i = 0; i < nx; i++) {
      for (int j = 0; j < nx; j++) g[i * nx + j] += lh[i] * x[j] + lam[i] * dx[j];
      for (int j = 0; j < nu; j++) g[nx * nx + i * nu + j] += lh[i] * u[j] + lam[i] * du[j];
    }
  } else if (md->kind == DIFFMPC_KIND_PLANAR_QUADROTOR) {
    double m = mp[0], arm = mp[1], I = mp[2];
    double s = sin(x[2]), c = cos(x[2]);
    double F = u[0] + u[1], dF = du[0] + du[1], dd = u[1] - u[0], ddd = du[1] - du[0];
    /* m: f3 = x3 - dt F s/m, f4 = x4 + dt (F c/m - g) */
    g[0] += lh[3] * (dt * F * s / (m * m)) + lh[4] * (-dt * F * c / (m * m))
          + lam[3] * (dt * (F * c * dx[2] + s * dF) / (m * m))
          + lam[4] * (dt * (F * s * dx[2] - c * dF) / (m * m));
    /* arm, inertia: f5 = x5 + dt arm (u1-u0)/I */
    g[1] += lh[5] * (dt * dd / I) + lam[5] * (dt * ddd / I);
    g[2] += lh[5] * (-dt * arm * dd / (I * I)) + lam[5] * (-dt * arm * ddd / (I * I));
    /* g: f4 -= dt g */
    g[3] += lh[4] * (-dt);
  } else if (md->kind == DIFFMPC_KIND_QUADROTOR13) {
    double m = mp[0], l = mp[1], Jx = mp[2], Jy = mp[3], Jz = mp[4], kap = mp[5];
    double d = l * INV_SQRT2;
    double qw = x[3], qx = x[4], qy = x[5], qz = x[6];
    double wx = x[10], wy = x[11], wz = x[12];
    double dqw = dx[3], dqx = dx[4], dqy = dx[5], dqz = dx[6];
    double dwx = dx[10], dwy = dx[11], dwz = dx[12];
    double F = ((u[0] + u[1]) + u[2]) + u[3];
    double dF = ((du[0] + du[1]) + du[2]) + du[3];
    double sx = ((u[0] + u[1]) - u[2]) - u[3], dsx = ((du[0] + du[1]) - du[2]) - du[3];
    double sy = ((u[1] - u[0]) + u[2]) - u[3], dsy = ((du[1] - du[0]) + du[2]) - du[3];
    double sz = ((u[0] - u[1]) + u[2]) - u[3], dsz = ((du[0] - du[1]) + du[2]) - du[3];
    double tx = d * sx, ty = d * sy, tz = kap * sz;
    double r13 = 2.0 * (qx * qz + qw * qy), r23 = 2.0 * (qy * qz - qw * qx);
    double r33 = 1.0 - 2.0 * (qx * qx + qy * qy);
    double dr13 = 2.0 * (qy * dqw + qz * dqx + qw * dqy + qx * dqz);
    double dr23 = 2.0 * (-qx * dqw - qw * dqx + qz * dqy + qy * dqz);
    double dr33 = -4.0 * (qx * dqx + qy * dqy);
    double im2 = dt / (m * m);
    /* m */
    g[0] += -im2 * F * (lh[7] * r13 + lh[8] * r23 + lh[9] * r33)
          - im2 * (lam[7] * (F * dr13 + r13 * dF) + lam[8] * (F * dr23 + r23 * dF) + lam[9] * (F * dr33 + r33 * dF));
    /* arm */
    g[1] += lh[10] * (dt * INV_SQRT2 * sx / Jx) + lh[11] * (dt * INV_SQRT2 * sy / Jy)
          + lam[10] * (dt * INV_SQRT2 * dsx / Jx) + lam[11] * (dt * INV_SQRT2 * dsy / Jy);
    /* Jx, Jy, Jz */
    double e10 = tx - (Jz - Jy) * wy * wz, e11 = ty - (Jx - Jz) * wz * wx, e12 = tz - (Jy - Jx) * wx * wy;
    double de10 = d * dsx - (Jz - Jy) * (wz * dwy + wy * dwz);
    double de11 = d * dsy - (Jx - Jz) * (wx * dwz + wz * dwx);
    double de12 = kap * dsz - (Jy - Jx) * (wy * dwx + wx * dwy);
    double pwz = wy * wz, pzx = wz * wx, pxy = wx * wy;
    double dpyz = wz * dwy + wy * dwz, dpzx = wx * dwz + wz * dwx, dpxy = wy * dwx + wx * dwy;
    g[2] += lh[10] * (-dt * e10 / (Jx * Jx)) + lh[11] * (-dt * pzx / Jy) + lh[12] * (dt * pxy / Jz)
          + lam[10] * (-dt * de10 / (Jx * Jx)) + lam[11] * (-dt * dpzx / Jy) + lam[12] * (dt * dpxy / Jz);
    g[3] += lh[10] * (dt * pwz / Jx) + lh[11] * (-dt * e11 / (Jy * Jy)) + lh[12] * (-dt * pxy / Jz)
          + lam[10] * (dt * dpyz / Jx) + lam[11] * (-dt * de11 / (Jy * Jy)) + lam[12] * (-dt * dpxy / Jz);
    g[4] += lh[10] * (-dt * pwz / Jx) + lh[11] * (dt * pzx / Jy) + lh[12] * (-dt * e12 / (Jz * Jz))
          + lam[10] * (-dt * dpyz / Jx) + lam[11] * (dt * dpzx / Jy) + lam[12] * (-dt * de12 / (Jz * Jz));
    /* kappa */
    g[5] += lh[12] * (dt * sz / Jz) + lam[12] * (dt * dsz / Jz);
    /* g */
    g[6] += lh[9] * (-dt);
  }
  /* double integrator: no parameters */
}

/* ------------------------------------------------------------------------- */
/* cost, Cholesky, box QP: kernels.py:120-318                                 */
/* ------------------------------------------------------------------------- */

/* _stage_cost_xu (kernels.py:133-145): i-outer, same accumulation order */
static double stage_cost_xu(const double* Ct, const double* ct, const double* x, const double* u, int nx, int nz) {
  double acc = 0.0;
  for (int i = 0; i < nz; i++) {
    double zi = i < nx ? x[i] : u[i - nx];
    double row = 0.0;
    for (int j = 0; j < nz; j++) {
      double zj = j < nx ? x[j] : u[j - nx];
      row += Ct[i * nz + j] * zj;
    }
    acc += 0.5 * zi * row + ct[i] * zi;
  }
  return acc;
}

static int finite_vec(const double* v, int n) {
  for (int i = 0; i < n; i++)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* _chol_factor (kernels.py:195-209): lower Cholesky of H[idx,idx]; H is (ld x ld) */
static int chol_factor(const double* H, int ld, double* L, const int* idx, int nf) {
  for (int a = 0; a < nf; a++) {
    for (int b = 0; b <= a; b++) {
      double s = H[idx[a] * ld + idx[b]];
      for (int r = 0; r < b; r++) s -= L[a * MAXN + r] * L[b * MAXN + r];
      if (a == b) {
        if (s <= 0.0) return 0;
        L[a * MAXN + a] = sqrt(s);
      } else {
        L[a * MAXN + b] = s / L[b * MAXN + b];
      }
    }
  }
  return 1;
}

/* _chol_solve (kernels.py:212-224) */
static void chol_solve(const double* L, const double* b, double* out, int nf) {
  for (int a = 0; a < nf; a++) {
    double s = b[a];
    for (int r = 0; r < a; r++) s -= L[a * MAXN + r] * out[r];
    out[a] = s / L[a * MAXN + a];
  }
  for (int a = nf - 1; a >= 0; a--) {
    double s = out[a];
    for (int r = a + 1; r < nf; r++) s -= L[r * MAXN + a] * out[r];
    out[a] = s / L[a * MAXN + a];
  }
}

/* _qp_value (kernels.py:227-236) */
static double qp_value(const double* H, const double* g, const double* u, int n) {
  double acc = 0.0;
  for (int a = 0; a < n; a++) {
    double row = 0.0;
    for (int b = 0; b < n; b++) row += H[a * n + b] * u[b];
    acc += 0.5 * u[a] * row + g[a] * u[a];
  }
  return acc;
}

/* boxqp_one (kernels.py:239-318): projected Newton with Armijo backtracking.
 * H (n x n), returns 0 ok / -1 not PD; free[] marks the last clamp detection. */
int oracle_boxqp(const double* H, const double* g, const double* lo, const double* hi, double* u,
                 uint8_t* free_, int n, int max_iter, double tol) {
  double L[MAXN * MAXN], grad[MAXN], search[MAXN], rhs[MAXN], cand[MAXN];
  int idx[MAXN];
  for (int a = 0; a < n; a++) {
    if (u[a] < lo[a]) u[a] = lo[a];
    else if (u[a] > hi[a]) u[a] = hi[a];
    free_[a] = 1;
  }
  double value = qp_value(H, g, u, n);
  for (int it = 0; it < max_iter; it++) {
    int n_free = 0;
    for (int a = 0; a < n; a++) {
      double s = g[a];
      for (int b = 0; b < n; b++) s += H[a * n + b] * u[b];
      grad[a] = s;
      int clamped = (u[a] <= lo[a] && s > 0.0) || (u[a] >= hi[a] && s < 0.0);
      if (clamped) {
        free_[a] = 0;
      } else {
        free_[a] = 1;
        idx[n_free++] = a;
      }
    }
    if (n_free == 0) return 0;
    double gnorm = 0.0;
    for (int a = 0; a < n_free; a++) gnorm += grad[idx[a]] * grad[idx[a]];
    if (sqrt(gnorm) <= tol) return 0;
    if (!chol_factor(H, n, L, idx, n_free)) return -1;
    for (int a = 0; a < n_free; a++) {
      double s = g[idx[a]];
      for (int b = 0; b < n; b++)
        if (free_[b] == 0) s += H[idx[a] * n + b] * u[b];
      rhs[a] = s;
    }
    chol_solve(L, rhs, cand, n_free);
    for (int a = 0; a < n; a++) search[a] = 0.0;
    double sdotg = 0.0;
    for (int a = 0; a < n_free; a++) {
      double st = -cand[a] - u[idx[a]];
      search[idx[a]] = st;
      sdotg += st * grad[idx[a]];
    }
    if (sdotg >= 0.0) return 0;
    double step = 1.0, vc = 0.0;
    int accepted = 0;
    while (step > MIN_STEP) {
      for (int a = 0; a < n; a++) {
        double v = u[a] + step * search[a];
        if (v < lo[a]) v = lo[a];
        else if (v > hi[a]) v = hi[a];
        cand[a] = v;
      }
      vc = qp_value(H, g, cand, n);
      if (vc - value <= ARMIJO * step * sdotg) { accepted = 1; break; }
      step *= STEP_DEC;
    }
    if (!accepted) return 0;
    for (int a = 0; a < n; a++) u[a] = cand[a];
    value = vc;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* per-instance forward solve: ilqr.run_staged_solve (ilqr.py:154-247)         */
/* ------------------------------------------------------------------------- */

typedef struct {
  const DiffMPCProblem* p;
  const DiffMPCForwardIO* io;
  const DiffMPCBackwardIO* bio;
  int lo, hi;
} Job;

static const double* theta_of(const DiffMPCProblem* p, const void* theta, int i) {
  return (const double*)theta + (size_t)p->theta_stride * i;
}

/* Expand (dense or diag) cost of instance i, stage t into a dense nz x nz block. */
static void load_C(const DiffMPCProblem* p, const double* C, int i, int t, double* out) {
  int nz = p->nx + p->nu;
  if (p->cost_layout == DIFFMPC_COST_DENSE) {
    memcpy(out, C + ((size_t)i * p->T + t) * nz * nz, sizeof(double) * nz * nz);
  } else {
    const double* d = C + ((size_t)i * p->T + t) * nz;
    for (int a = 0; a < nz * nz; a++) out[a] = 0.0;
    for (int a = 0; a < nz; a++) out[a * nz + a] = d[a];
  }
}

static void solve_instance(const DiffMPCProblem* p, const DiffMPCForwardIO* io, int i) {
  const int T = p->T, nx = p->nx, nu = p->nu, nz = nx + nu, na = p->n_alpha;
  Model md = {p->model_kind, nx, nu, p->dt, theta_of(p, io->theta, i)};
  const double* Cin = (const double*)io->C;
  const double* cin = (const double*)io->c + (size_t)i * T * nz;
  /* workspace (Workspace, ilqr.py:84-113), one instance */
  double* Call = (double*)malloc(sizeof(double) * T * nz * nz);
  double* X = (double*)calloc((size_t)(T + 1) * nx, sizeof(double));
  double* U = (double*)calloc((size_t)T * nu, sizeof(double));
  double* A = (double*)calloc((size_t)T * nx * nx, sizeof(double));
  double* Bm = (double*)calloc((size_t)T * nx * nu, sizeof(double));
  double* K = (double*)calloc((size_t)T * nu * nx, sizeof(double));
  double* k = (double*)calloc((size_t)T * nu, sizeof(double));
  double* Xc = (double*)calloc((size_t)na * (T + 1) * nx, sizeof(double));
  double* Uc = (double*)calloc((size_t)na * T * nu, sizeof(double));
  for (int t = 0; t < T; t++) load_C(p, Cin, i, t, Call + (size_t)t * nz * nz);
  const double* umin = p->u_min;
  const double* umax = p->u_max;
  memcpy(X, (const double*)io->x0 + (size_t)i * nx, sizeof(double) * nx);
  memcpy(U, (const double*)io->U_warm + (size_t)i * T * nu, sizeof(double) * T * nu);
  /* np.clip(ws.U, u_min, u_max) (ilqr.py:165) */
  for (int t = 0; t < T; t++)
    for (int r = 0; r < nu; r++) {
      double v = U[t * nu + r];
      v = v < umin[r] ? umin[r] : v;
      v = v > umax[r] ? umax[r] : v;
      U[t * nu + r] = v;
    }
  int active = 1, fail_t = -1, iterations = 0, converged = 0, diverged = 0;
  double J = 0.0;
  double* ah = io->alpha_hist ? (double*)io->alpha_hist + (size_t)i * p->K_max : NULL;
  double* Jh = io->J_hist ? (double*)io->J_hist + (size_t)i * (p->K_max + 1) : NULL;
  if (ah) for (int it = 0; it < p->K_max; it++) ah[it] = 0.0;
  /* initial rollout (kernels.py:161-178) */
  for (int t = 0; t < T; t++) {
    J += stage_cost_xu(Call + (size_t)t * nz * nz, cin + t * nz, X + t * nx, U + t * nu, nx, nz);
    step_one(&md, X + t * nx, U + t * nu, X + (t + 1) * nx);
    if (!finite_vec(X + (t + 1) * nx, nx)) {
      fail_t = t; active = 0; J = INFINITY;
      break;
    }
  }
  if (fail_t >= 0) diverged = 1; /* rollout_failed (ilqr.py:196-200) */
  if (Jh) Jh[0] = J;
  double Vx[MAXN], Vxx[MAXN * MAXN];
  double gz[MAXN], qx[MAXN], qu[MAXN], qxx[MAXN * MAXN], qux[MAXN * MAXN], quu[MAXN * MAXN];
  double quu_try[MAXN * MAXN], MA[MAXN * MAXN], NB[MAXN * MAXN], lo[MAXN], hi[MAXN], du[MAXN];
  double L[MAXN * MAXN], rhs[MAXN], kcol[MAXN], newVx[MAXN], newVxx[MAXN * MAXN];
  double Jc[DIFFMPC_MAX_ALPHA];
  uint8_t freem[MAXN], dead[DIFFMPC_MAX_ALPHA];
  int idx[MAXN];
  int it;
  for (it = 0; it < p->K_max; it++) {
    if (!active) break;
    /* stage 1: linearize (kernels.py:181-187) */
    for (int t = 0; t < T; t++) jac_one(&md, X + t * nx, U + t * nu, A + t * nx * nx, Bm + t * nx * nu);
    /* stage 2: Riccati sweep (kernels.py:326-512); Vx = Vxx = 0 (ilqr.py:208-209) */
    for (int a = 0; a < nx; a++) Vx[a] = 0.0;
    for (int a = 0; a < nx * nx; a++) Vxx[a] = 0.0;
    for (int t = T - 1; t >= 0; t--) {
      const double* At = A + t * nx * nx;
      const double* Bt = Bm + t * nx * nu;
      const double* Ct = Call + (size_t)t * nz * nz;
      const double* ct = cin + t * nz;
      const double* x = X + t * nx;
      const double* u = U + t * nu;
      for (int a = 0; a < nz; a++) {
        double s = ct[a];
        for (int b = 0; b < nz; b++) s += Ct[a * nz + b] * (b < nx ? x[b] : u[b - nx]);
        gz[a] = s;
      }
      for (int a = 0; a < nx; a++) {
        double s = gz[a];
        for (int b = 0; b < nx; b++) s += At[b * nx + a] * Vx[b];
        qx[a] = s;
      }
      for (int a = 0; a < nu; a++) {
        double s = gz[nx + a];
        for (int b = 0; b < nx; b++) s += Bt[b * nu + a] * Vx[b];
        qu[a] = s;
      }
      for (int a = 0; a < nx; a++) {
        for (int b = 0; b < nx; b++) {
          double s = 0.0;
          for (int r = 0; r < nx; r++) s += Vxx[a * nx + r] * At[r * nx + b];
          MA[a * nx + b] = s;
        }
        for (int b = 0; b < nu; b++) {
          double s = 0.0;
          for (int r = 0; r < nx; r++) s += Vxx[a * nx + r] * Bt[r * nu + b];
          NB[a * nu + b] = s;
        }
      }
      for (int a = 0; a < nx; a++)
        for (int b = 0; b < nx; b++) {
          double s = Ct[a * nz + b];
          for (int r = 0; r < nx; r++) s += At[r * nx + a] * MA[r * nx + b];
          qxx[a * nx + b] = s;
        }
      for (int a = 0; a < nu; a++)
        for (int b = 0; b < nx; b++) {
          double s = Ct[(nx + a) * nz + b];
          for (int r = 0; r < nx; r++) s += Bt[r * nu + a] * MA[r * nx + b];
          qux[a * nx + b] = s;
        }
      for (int a = 0; a < nu; a++)
        for (int b = 0; b < nu; b++) {
          double s = Ct[(nx + a) * nz + nx + b];
          for (int r = 0; r < nx; r++) s += Bt[r * nu + a] * NB[r * nu + b];
          quu[a * nu + b] = s;
        }
      for (int a = 0; a < nu; a++) {
        lo[a] = umin[a] - u[a];
        hi[a] = umax[a] - u[a];
      }
      /* lambda schedule (kernels.py:444-471) */
      double lam = 0.0;
      int ok = 0;
      for (;;) {
        for (int a = 0; a < nu; a++)
          for (int b = 0; b < nu; b++) quu_try[a * nu + b] = quu[a * nu + b] + (a == b ? lam : 0.0);
        for (int a = 0; a < nu; a++) du[a] = 0.0;
        int st = oracle_boxqp(quu_try, qu, lo, hi, du, freem, nu, p->boxqp_max_iter, p->boxqp_tol);
        if (st == 0) {
          int nf = 0;
          for (int a = 0; a < nu; a++)
            if (freem[a] == 1) idx[nf++] = a;
          if (nf == 0 || chol_factor(quu_try, nu, L, idx, nf)) { ok = 1; break; }
        }
        lam = lam == 0.0 ? LAM_INIT : lam * 10.0;
        if (lam > LAM_MAX) break;
      }
      if (!ok) { fail_t = t; active = 0; break; }
      int nf = 0;
      for (int a = 0; a < nu; a++) {
        if (freem[a] == 1) idx[nf++] = a;
        k[t * nu + a] = du[a];
        for (int b = 0; b < nx; b++) K[(t * nu + a) * nx + b] = 0.0;
      }
      for (int col = 0; col < nx && nf > 0; col++) {
        for (int a = 0; a < nf; a++) rhs[a] = qux[idx[a] * nx + col];
        chol_solve(L, rhs, kcol, nf);
        for (int a = 0; a < nf; a++) K[(t * nu + idx[a]) * nx + col] = -kcol[a];
      }
      const double* Kt = K + t * nu * nx;
      const double* kt = k + t * nu;
      for (int a = 0; a < nx; a++) {
        double s = qx[a];
        for (int r = 0; r < nu; r++) {
          double rowq = 0.0;
          for (int b = 0; b < nu; b++) rowq += quu[r * nu + b] * kt[b];
          s += Kt[r * nx + a] * (rowq + qu[r]) + qux[r * nx + a] * kt[r];
        }
        newVx[a] = s;
      }
      for (int a = 0; a < nx; a++)
        for (int b = 0; b < nx; b++) {
          double s = qxx[a * nx + b];
          for (int r = 0; r < nu; r++) {
            double rowq = 0.0;
            for (int q2 = 0; q2 < nu; q2++) rowq += quu[r * nu + q2] * Kt[q2 * nx + b];
            s += Kt[r * nx + a] * rowq + Kt[r * nx + a] * qux[r * nx + b] + qux[r * nx + a] * Kt[r * nx + b];
          }
          newVxx[a * nx + b] = s;
        }
      for (int a = 0; a < nx; a++) Vx[a] = newVx[a];
      for (int a = 0; a < nx; a++)
        for (int b = 0; b < nx; b++) Vxx[a * nx + b] = 0.5 * (newVxx[a * nx + b] + newVxx[b * nx + a]);
    }
    /* stage 3: line search (kernels.py:520-574), candidates reset (ilqr.py:211-213) */
    for (int a = 0; a < na; a++) {
      Jc[a] = 0.0;
      dead[a] = 0;
      memcpy(Xc + (size_t)a * (T + 1) * nx, X, sizeof(double) * nx);
    }
    if (active) {
      for (int a = 0; a < na; a++) {
        double alpha = p->alphas[a];
        double* xca = Xc + (size_t)a * (T + 1) * nx;
        double* uca = Uc + (size_t)a * T * nu;
        for (int t = 0; t < T; t++) {
          const double* xc = xca + t * nx;
          for (int r = 0; r < nu; r++) {
            double v = U[t * nu + r] + alpha * k[t * nu + r];
            for (int b = 0; b < nx; b++) v += K[(t * nu + r) * nx + b] * (xc[b] - X[t * nx + b]);
            if (v < umin[r]) v = umin[r];
            else if (v > umax[r]) v = umax[r];
            uca[t * nu + r] = v;
          }
          Jc[a] += stage_cost_xu(Call + (size_t)t * nz * nz, cin + t * nz, xc, uca + t * nu, nx, nz);
          step_one(&md, xc, uca + t * nu, xca + (t + 1) * nx);
          if (!finite_vec(xca + (t + 1) * nx, nx) || !isfinite(Jc[a])) {
            dead[a] = 1;
            Jc[a] = INFINITY;
            break;
          }
        }
      }
    }
    /* epilogue (ilqr.py:216-244) */
    int act = active;
    if (act) iterations = it + 1;
    int best = 0;
    for (int a = 1; a < na; a++)
      if (Jc[a] < Jc[best]) best = a; /* np.argmin: first minimum */
    double best_J = Jc[best];
    int alld = 1;
    for (int a = 0; a < na; a++) alld &= dead[a];
    int all_dead = act && alld;
    int accept = act && !all_dead && (best_J < J);
    if (ah) ah[it] = accept ? p->alphas[best] : 0.0;
    if (accept) {
      memcpy(X, Xc + (size_t)best * (T + 1) * nx, sizeof(double) * (T + 1) * nx);
      memcpy(U, Uc + (size_t)best * T * nu, sizeof(double) * T * nu);
    }
    double J_prev = J;
    if (accept) J = best_J;
    if (all_dead) { diverged = 1; active = 0; }
    double rel = fabs(J_prev - J) / fmax(1.0, fabs(J_prev));
    int no_step = act && !all_dead && !accept;
    int conv_now = (act && !all_dead) && (no_step || rel <= p->conv_tol);
    if (conv_now) { converged = 1; active = 0; }
    if (Jh) Jh[it + 1] = J;
  }
  if (Jh)
    for (int j = it + 1; j <= p->K_max; j++) Jh[j] = J;
  /* collect_result (ilqr.py:250-268) */
  int failed = fail_t >= 0 || diverged;
  memcpy((double*)io->X + (size_t)i * (T + 1) * nx, X, sizeof(double) * (T + 1) * nx);
  memcpy((double*)io->U + (size_t)i * T * nu, U, sizeof(double) * T * nu);
  ((double*)io->J)[i] = J;
  if (io->K) memcpy((double*)io->K + (size_t)i * T * nu * nx, K, sizeof(double) * T * nu * nx);
  if (io->k) memcpy((double*)io->k + (size_t)i * T * nu, k, sizeof(double) * T * nu);
  if (io->iters) io->iters[i] = iterations;
  if (io->converged) io->converged[i] = (uint8_t)(converged && !failed);
  if (io->diverged) io->diverged[i] = (uint8_t)diverged;
  if (io->fail_t) io->fail_t[i] = fail_t;
  if (io->clamped)
    for (int t = 0; t < T; t++)
      for (int r = 0; r < nu; r++)
        io->clamped[((size_t)i * T + t) * nu + r] = (uint8_t)(U[t * nu + r] <= umin[r] || U[t * nu + r] >= umax[r]);
  free(Call); free(X); free(U); free(A); free(Bm); free(K); free(k); free(Xc); free(Uc);
}

/* ------------------------------------------------------------------------- */
/* per-instance implicit backward: policy.py:257-283 + gradlayer.py:98-150 +    */
/* kernels.py:582-756, plus the NEW dtheta / dL/dJ adjoint terms               */
/* ------------------------------------------------------------------------- */

static void backward_instance(const DiffMPCProblem* p, const DiffMPCBackwardIO* io, int i) {
  const int T = p->T, nx = p->nx, nu = p->nu, nz = nx + nu;
  Model md = {p->model_kind, nx, nu, p->dt, theta_of(p, io->theta, i)};
  const double* X = (const double*)io->X + (size_t)i * (T + 1) * nx;
  const double* U = (const double*)io->U + (size_t)i * T * nu;
  const double* sX = io->dLdX ? (const double*)io->dLdX + (size_t)i * (T + 1) * nx : NULL;
  const double* sU = io->dLdU ? (const double*)io->dLdU + (size_t)i * T * nu : NULL;
  double sJ = io->dLdJ ? ((const double*)io->dLdJ)[i] : 0.0;
  double* Call = (double*)malloc(sizeof(double) * T * nz * nz);
  double* A = (double*)malloc(sizeof(double) * T * nx * nx);
  double* Bm = (double*)malloc(sizeof(double) * T * nx * nu);
  double* K = (double*)calloc((size_t)T * nu * nx, sizeof(double));
  double* k = (double*)calloc((size_t)T * nu, sizeof(double));
  double* dX = (double*)calloc((size_t)(T + 1) * nx, sizeof(double));
  double* dU = (double*)calloc((size_t)T * nu, sizeof(double));
  double* dC = (double*)calloc((size_t)T * nz * nz, sizeof(double));
  double* dc = (double*)calloc((size_t)T * nz, sizeof(double));
  uint8_t* clamped = (uint8_t*)malloc((size_t)T * nu);
  for (int t = 0; t < T; t++) load_C(p, (const double*)io->C, i, t, Call + (size_t)t * nz * nz);
  /* relinearize at the final (X,U), all instances active (policy.py:257-267) */
  for (int t = 0; t < T; t++) jac_one(&md, X + t * nx, U + t * nu, A + t * nx * nx, Bm + t * nx * nu);
  /* clamped = (U<=u_min)|(U>=u_max) (policy.py:271) */
  for (int t = 0; t < T; t++)
    for (int r = 0; r < nu; r++)
      clamped[t * nu + r] = (uint8_t)(U[t * nu + r] <= p->u_min[r] || U[t * nu + r] >= p->u_max[r]);
  /* run_staged_backward init (gradlayer.py:106-110) */
  double Vx[MAXN], Vxx[MAXN * MAXN];
  for (int a = 0; a < nx; a++) Vx[a] = sX ? sX[T * nx + a] : 0.0;
  for (int a = 0; a < nx * nx; a++) Vxx[a] = 0.0;
  int fail_t = -1;
  double qx[MAXN], qu[MAXN], qxx[MAXN * MAXN], qux[MAXN * MAXN], quu[MAXN * MAXN];
  double MA[MAXN * MAXN], NB[MAXN * MAXN], L[MAXN * MAXN], rhs[MAXN], sol[MAXN];
  double newVx[MAXN], newVxx[MAXN * MAXN];
  int idx[MAXN];
  /* aux_backward_range (kernels.py:582-707) */
  for (int t = T - 1; t >= 0; t--) {
    const double* At = A + t * nx * nx;
    const double* Bt = Bm + t * nx * nu;
    const double* Ct = Call + (size_t)t * nz * nz;
    for (int a = 0; a < nx; a++) {
      double s = sX ? sX[t * nx + a] : 0.0;
      for (int b = 0; b < nx; b++) s += At[b * nx + a] * Vx[b];
      qx[a] = s;
    }
    for (int a = 0; a < nu; a++) {
      double s = sU ? sU[t * nu + a] : 0.0;
      for (int b = 0; b < nx; b++) s += Bt[b * nu + a] * Vx[b];
      qu[a] = s;
    }
    for (int a = 0; a < nx; a++) {
      for (int b = 0; b < nx; b++) {
        double s = 0.0;
        for (int r = 0; r < nx; r++) s += Vxx[a * nx + r] * At[r * nx + b];
        MA[a * nx + b] = s;
      }
      for (int b = 0; b < nu; b++) {
        double s = 0.0;
        for (int r = 0; r < nx; r++) s += Vxx[a * nx + r] * Bt[r * nu + b];
        NB[a * nu + b] = s;
      }
    }
    for (int a = 0; a < nx; a++)
      for (int b = 0; b < nx; b++) {
        double s = Ct[a * nz + b];
        for (int r = 0; r < nx; r++) s += At[r * nx + a] * MA[r * nx + b];
        qxx[a * nx + b] = s;
      }
    for (int a = 0; a < nu; a++)
      for (int b = 0; b < nx; b++) {
        double s = Ct[(nx + a) * nz + b];
        for (int r = 0; r < nx; r++) s += Bt[r * nu + a] * MA[r * nx + b];
        qux[a * nx + b] = s;
      }
    for (int a = 0; a < nu; a++)
      for (int b = 0; b < nu; b++) {
        double s = Ct[(nx + a) * nz + nx + b];
        for (int r = 0; r < nx; r++) s += Bt[r * nu + a] * NB[r * nu + b];
        quu[a * nu + b] = s;
      }
    for (int a = 0; a < nu; a++) {
      if (clamped[t * nu + a] == 1) {
        qu[a] = 0.0;
        for (int b = 0; b < nx; b++) qux[a * nx + b] = 0.0;
        for (int b = 0; b < nu; b++) { quu[a * nu + b] = 0.0; quu[b * nu + a] = 0.0; }
        quu[a * nu + a] = 1.0;
      }
    }
    for (int a = 0; a < nu; a++) idx[a] = a;
    if (!chol_factor(quu, nu, L, idx, nu)) { fail_t = t; break; }
    for (int a = 0; a < nu; a++) rhs[a] = qu[a];
    chol_solve(L, rhs, sol, nu);
    for (int a = 0; a < nu; a++) k[t * nu + a] = -sol[a];
    for (int col = 0; col < nx; col++) {
      for (int a = 0; a < nu; a++) rhs[a] = qux[a * nx + col];
      chol_solve(L, rhs, sol, nu);
      for (int a = 0; a < nu; a++) K[(t * nu + a) * nx + col] = -sol[a];
    }
    const double* Kt = K + t * nu * nx;
    const double* kt = k + t * nu;
    for (int a = 0; a < nx; a++) {
      double s = qx[a];
      for (int r = 0; r < nu; r++) {
        double rowq = 0.0;
        for (int b = 0; b < nu; b++) rowq += quu[r * nu + b] * kt[b];
        s += Kt[r * nx + a] * (rowq + qu[r]) + qux[r * nx + a] * kt[r];
      }
      newVx[a] = s;
    }
    for (int a = 0; a < nx; a++)
      for (int b = 0; b < nx; b++) {
        double s = qxx[a * nx + b];
        for (int r = 0; r < nu; r++) {
          double rowq = 0.0;
          for (int q2 = 0; q2 < nu; q2++) rowq += quu[r * nu + q2] * Kt[q2 * nx + b];
          s += Kt[r * nx + a] * rowq + Kt[r * nx + a] * qux[r * nx + b] + qux[r * nx + a] * Kt[r * nx + b];
        }
        newVxx[a * nx + b] = s;
      }
    for (int a = 0; a < nx; a++) Vx[a] = newVx[a];
    for (int a = 0; a < nx; a++)
      for (int b = 0; b < nx; b++) Vxx[a * nx + b] = 0.5 * (newVxx[a * nx + b] + newVxx[b * nx + a]);
  }
  int n_theta = p->n_theta;
  double gth[2048];
  for (int j = 0; j < n_theta && j < 2048; j++) gth[j] = 0.0;
  if (fail_t < 0) {
    /* aux_rollout_range (kernels.py:710-730) */
    for (int t = 0; t < T; t++) {
      for (int r = 0; r < nu; r++) {
        double s = k[t * nu + r];
        for (int b = 0; b < nx; b++) s += K[(t * nu + r) * nx + b] * dX[t * nx + b];
        dU[t * nu + r] = s;
      }
      for (int a = 0; a < nx; a++) {
        double s = 0.0;
        for (int b = 0; b < nx; b++) s += A[t * nx * nx + a * nx + b] * dX[t * nx + b];
        for (int b = 0; b < nu; b++) s += Bm[t * nx * nu + a * nu + b] * dU[t * nu + b];
        dX[(t + 1) * nx + a] = s;
      }
    }
    /* aux_assemble_range (kernels.py:733-756) */
    for (int t = 0; t < T; t++) {
      for (int a = 0; a < nz; a++) {
        double da = a < nx ? dX[t * nx + a] : dU[t * nu + a - nx];
        dc[t * nz + a] = da;
        double za = a < nx ? X[t * nx + a] : U[t * nu + a - nx];
        for (int b = 0; b < nz; b++) {
          double db = b < nx ? dX[t * nx + b] : dU[t * nu + b - nx];
          double zb = b < nx ? X[t * nx + b] : U[t * nu + b - nx];
          dC[(t * nz + a) * nz + b] = 0.5 * (da * zb + za * db);
        }
      }
      for (int a = 0; a < nu; a++) {
        if (clamped[t * nu + a] == 1) {
          dc[t * nz + nx + a] = 0.0;
          for (int b = 0; b < nz; b++) {
            dC[(t * nz + nx + a) * nz + b] = 0.0;
            dC[(t * nz + b) * nz + nx + a] = 0.0;
          }
        }
      }
    }
    /* NEW: primal co-state lam and aux co-state lh, backward in t.
     * lam_T = 0,       lam_t = [C_t z_t + c_t]_x + A_t' lam_{t+1}
     * lh_T = dL/dX_T,  lh_t  = dL/dX_t + [C_t dz_t]_x + A_t' lh_{t+1}
     * dtheta = sum_t lh_{t+1}' df/dth + lam_{t+1}' (d2f/dth dz) dz_t ;
     * optimal-cost (envelope) terms scaled by dL/dJ:
     * dC += sJ/2 z z', dc += sJ z, dx0 += sJ lam_0, dtheta += sJ sum_t lam_{t+1}' df/dth */
    const double* cc = (const double*)io->c + (size_t)i * T * nz;
    double lam[MAXN], lh[MAXN], nl[MAXN], nlh[MAXN], zero[MAXN];
    for (int a = 0; a < nx; a++) { lam[a] = 0.0; lh[a] = sX ? sX[T * nx + a] : 0.0; zero[a] = 0.0; }
    for (int t = T - 1; t >= 0; t--) {
      const double* x = X + t * nx;
      const double* u = U + t * nu;
      const double* Ct = Call + (size_t)t * nz * nz;
      /* dtheta uses lam_{t+1}, lh_{t+1} (current values) */
      if (n_theta > 0 && io->dtheta) {
        theta_grad_stage(&md, x, u, dX + t * nx, dU + t * nu, lh, lam, gth);
        if (sJ != 0.0) {
          double lsc[MAXN];
          for (int a = 0; a < nx; a++) lsc[a] = sJ * lam[a];
          theta_grad_stage(&md, x, u, zero, zero, lsc, zero, gth);
        }
      }
      for (int a = 0; a < nx; a++) {
        double s1 = cc[t * nz + a], s2 = sX ? sX[t * nx + a] : 0.0;
        for (int b = 0; b < nz; b++) {
          double zb = b < nx ? x[b] : u[b - nx];
          double db = b < nx ? dX[t * nx + b] : dU[t * nu + b - nx];
          s1 += Ct[a * nz + b] * zb;
          s2 += Ct[a * nz + b] * db;
        }
        for (int b = 0; b < nx; b++) {
          s1 += A[t * nx * nx + b * nx + a] * lam[b];
          s2 += A[t * nx * nx + b * nx + a] * lh[b];
        }
        nl[a] = s1;
        nlh[a] = s2;
      }
      for (int a = 0; a < nx; a++) { lam[a] = nl[a]; lh[a] = nlh[a]; }
      if (sJ != 0.0) {
        for (int a = 0; a < nz; a++) {
          double za = a < nx ? x[a] : u[a - nx];
          dc[t * nz + a] += sJ * za;
          for (int b = 0; b < nz; b++) {
            double zb = b < nx ? x[b] : u[b - nx];
            dC[(t * nz + a) * nz + b] += 0.5 * sJ * za * zb;
          }
        }
      }
    }
    if (sJ != 0.0)
      for (int a = 0; a < nx; a++) Vx[a] += sJ * lam[a];
  }
  /* outputs; failed instances get zero gradients (gradlayer.py:153-159, policy.py:277-280) */
  int failed = fail_t >= 0;
  if (io->dC) {
    if (p->cost_layout == DIFFMPC_COST_DENSE) {
      double* o = (double*)io->dC + (size_t)i * T * nz * nz;
      for (int j = 0; j < T * nz * nz; j++) o[j] = failed ? 0.0 : dC[j];
    } else {
      double* o = (double*)io->dC + (size_t)i * T * nz;
      for (int t = 0; t < T; t++)
        for (int a = 0; a < nz; a++) o[t * nz + a] = failed ? 0.0 : dC[(t * nz + a) * nz + a];
    }
  }
  if (io->dc) {
    double* o = (double*)io->dc + (size_t)i * T * nz;
    for (int j = 0; j < T * nz; j++) o[j] = failed ? 0.0 : dc[j];
  }
  if (io->dx0) {
    double* o = (double*)io->dx0 + (size_t)i * nx;
    for (int a = 0; a < nx; a++) o[a] = failed ? 0.0 : Vx[a];
  }
  if (io->dtheta && n_theta > 0) {
    double* o = (double*)io->dtheta + (size_t)i * n_theta;
    for (int j = 0; j < n_theta; j++) o[j] = failed ? 0.0 : gth[j];
  }
  if (io->dX) memcpy((double*)io->dX + (size_t)i * (T + 1) * nx, dX, sizeof(double) * (T + 1) * nx);
  if (io->dU) memcpy((double*)io->dU + (size_t)i * T * nu, dU, sizeof(double) * T * nu);
  if (io->fail_t) io->fail_t[i] = fail_t;
  free(Call); free(A); free(Bm); free(K); free(k); free(dX); free(dU); free(dC); free(dc); free(clamped);
}

/* ------------------------------------------------------------------------- */
/* batch drivers (thread pool over instances, like WorkerPool.parallel_for)   */
/* ------------------------------------------------------------------------- */

static void* fwd_worker(void* arg) {
  Job* j = (Job*)arg;
  for (int i = j->lo; i < j->hi; i++) solve_instance(j->p, j->io, i);
  return NULL;
}

static void* bwd_worker(void* arg) {
  Job* j = (Job*)arg;
  for (int i = j->lo; i < j->hi; i++) backward_instance(j->p, j->bio, i);
  return NULL;
}

static int check(const DiffMPCProblem* p) {
  if (p->T < 1 || p->nx < 1 || p->nu < 1 || p->nx + p->nu > MAXN) return -1;
  if (p->nu > DIFFMPC_MAX_NU || p->n_alpha < 1 || p->n_alpha > DIFFMPC_MAX_ALPHA) return -1;
  if (p->n_theta > 2048) return -1;
  return 0;
}

static void run_pool(void* (*fn)(void*), const DiffMPCProblem* p, const DiffMPCForwardIO* io,
                     const DiffMPCBackwardIO* bio, int nthreads) {
  int B = p->B;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > B) nthreads = B;
  if (nthreads <= 1) {
    Job j = {p, io, bio, 0, B};
    fn(&j);
    return;
  }
  pthread_t th[256];
  Job jobs[256];
  if (nthreads > 256) nthreads = 256;
  int chunk = (B + nthreads - 1) / nthreads;
  int n = 0;
  for (int lo = 0; lo < B; lo += chunk) {
    jobs[n].p = p; jobs[n].io = io; jobs[n].bio = bio;
    jobs[n].lo = lo; jobs[n].hi = lo + chunk < B ? lo + chunk : B;
    pthread_create(&th[n], NULL, fn, &jobs[n]);
    n++;
  }
  for (int j = 0; j < n; j++) pthread_join(th[j], NULL);
}

int oracle_forward(const DiffMPCProblem* p, const DiffMPCForwardIO* io, int nthreads) {
  if (check(p)) return -1;
  if (p->B <= 0) return 0;
  run_pool(fwd_worker, p, io, NULL, nthreads);
  return 0;
}

int oracle_backward(const DiffMPCProblem* p, const DiffMPCBackwardIO* io, int nthreads) {
  if (check(p)) return -1;
  if (p->B <= 0) return 0;
  run_pool(bwd_worker, p, NULL, io, nthreads);
  return 0;
}

/* batched step + Jacobians (kernels.py:43-117) */
int oracle_dynamics(const DiffMPCProblem* p, int N, const double* theta, const double* x, const double* u,
                    double* xn, double* A, double* Bm) {
  if (check(p)) return -1;
  int nx = p->nx, nu = p->nu;
  for (int i = 0; i < N; i++) {
    Model md = {p->model_kind, nx, nu, p->dt, theta + (size_t)p->theta_stride * i};
    if (xn) step_one(&md, x + (size_t)i * nx, u + (size_t)i * nu, xn + (size_t)i * nx);
    if (A && Bm) jac_one(&md, x + (size_t)i * nx, u + (size_t)i * nu, A + (size_t)i * nx * nx, Bm + (size_t)i * nx * nu);
  }
  return 0;
}

// models.cuh — dynamics models for the B200 DiffMPC kernels.
//
// Each model is a stateless trait with compile-time dimensions and templated
// device functions, so the same model code runs in float (Riccati / backward,
// f32 mode) and double (trajectory rollouts and cost evaluation).
//
//   step(th, dt, x, u, out)            x+ = f(x,u)           (kernels.py:43-73)
//   jac_const(th, dt, A, lda, B, l, G) every entry of A = df/dx, B = df/du that
//                                      does not depend on (x,u) (zeros, ones, dt
//                                      terms, constant mixer rows) — written once
//                                      per kernel, cooperatively by the G lanes
//   jac_vary(th, dt, x, u, A, lda, B)  the state-dependent entries only, rewritten
//                                      every stage (kernels.py:76-117)
//   theta_grad(...)                    dL/dtheta contributions of one stage
//                                      (SURVEY.md §8(a) NEW row)
//
// `th` is the model's PREPARED parameter array (prep(): the raw parameters followed by
// derived constants such as 1/m, 1/J, arm/sqrt(2)), so divisions by parameters become
// multiplications (<= 1 ulp from the reference's divisions). Expression trees otherwise
// follow oracle/diffmpc_oracle.c. The linear model keeps [A|B] in shared memory.
#pragma once
#include <cuda_runtime.h>

namespace dmpc {

#define DMPC_DEV __device__ __forceinline__

constexpr double kInvSqrt2 = 0.7071067811865476;

// ---------------------------------------------------------------------------
// double integrator, d = NU (kernels.py:47-51, 85-91)
// ---------------------------------------------------------------------------
template <int D>
struct DoubleIntegrator {
  static constexpr int NX = 2 * D, NU = D, NTH = 0, NP = 1, KIND = 0;
  static constexpr bool kLinearParams = false;
  template <class S>
  DMPC_DEV static void prep(const S*, S* P) { P[0] = S(0); }
  // structural nonzeros of A = df/dx and B = df/du (compile-time; zero terms are skipped)
  __host__ __device__ static constexpr bool a_nz(int r, int c) { return r == c || (r < D && c == r + D); }
  // entries that are the constant 1 (A = I + dt df/dx: the diagonal) or exactly dt
  __host__ __device__ static constexpr bool a_one(int r, int c) { return r == c; }
  __host__ __device__ static constexpr bool a_dt(int r, int c) { return r < D && c == r + D; }
  __host__ __device__ static constexpr bool b_nz(int r, int c) { return r >= D && r - D == c; }
  template <class S>
  DMPC_DEV static void step(const S*, S dt, const S* x, const S* u, S* o) {
#pragma unroll
    for (int i = 0; i < D; i++) {
      o[i] = x[i] + dt * x[D + i];
      o[D + i] = x[D + i] + dt * u[i];
    }
  }
  template <class S>
  DMPC_DEV static void jac_const(const S*, S dt, S* A, int lda, S* B, int ldb, int lane, int G) {
    for (int e = lane; e < NX * NX; e += G) {
      int i = e / NX, j = e % NX;
      A[i * lda + j] = (i == j) ? S(1) : ((i < D && j == i + D) ? dt : S(0));
    }
    for (int e = lane; e < NX * NU; e += G) {
      int i = e / NU, j = e % NU;
      B[i * ldb + j] = (i >= D && i - D == j) ? dt : S(0);
    }
  }
  template <class S>
  DMPC_DEV static void jac_vary(const S*, S, const S*, const S*, S*, int, S*, int) {}
  template <class S>
  DMPC_DEV static void theta_grad(const S*, S, const S*, const S*, const S*, const S*, const S*,
                                  const S*, S*) {}
};

// ---------------------------------------------------------------------------
// planar quadrotor, x = [px, py, theta, vx, vy, omega], u = [u_left, u_right],
// th = [m, arm, I, g] (dynamics.py:57-70, kernels.py:52-65, 92-111)
// ---------------------------------------------------------------------------
struct PlanarQuad {
  static constexpr int NX = 6, NU = 2, NTH = 4, NP = 6, KIND = 1;
  static constexpr bool kLinearParams = false;
  __host__ __device__ static constexpr bool a_nz(int r, int c) {
    return r == c || (r < 3 && c == r + 3) || ((r == 3 || r == 4) && c == 2);
  }
  __host__ __device__ static constexpr bool b_nz(int r, int c) { return r >= 3 && c >= 0; }
  __host__ __device__ static constexpr bool a_one(int r, int c) { return r == c; }
  __host__ __device__ static constexpr bool a_dt(int r, int c) { return r < 3 && c == r + 3; }
  // P = [m, arm, I, g, 1/m, arm/I]
  template <class S>
  DMPC_DEV static void prep(const S* th, S* P) {
    P[0] = th[0]; P[1] = th[1]; P[2] = th[2]; P[3] = th[3];
    P[4] = S(1) / th[0];
    P[5] = th[1] / th[2];
  }
  template <class S>
  DMPC_DEV static void step(const S* P, S dt, const S* x, const S* u, S* o) {
    const S g = P[3], im = P[4], aoi = P[5];
    S s, c;
    sincos_(x[2], &s, &c);
    const S thrust = u[0] + u[1];
    o[0] = x[0] + dt * x[3];
    o[1] = x[1] + dt * x[4];
    o[2] = x[2] + dt * x[5];
    o[3] = x[3] + dt * (-thrust * s * im);
    o[4] = x[4] + dt * (thrust * c * im - g);
    o[5] = x[5] + dt * ((u[1] - u[0]) * aoi);
  }
  template <class S>
  DMPC_DEV static void jac_const(const S* P, S dt, S* A, int lda, S* B, int ldb, int lane, int G) {
    for (int e = lane; e < NX * NX; e += G) {
      int i = e / NX, j = e % NX;
      A[i * lda + j] = (i == j) ? S(1) : ((i < 3 && j == i + 3) ? dt : S(0));
    }
    for (int e = lane; e < NX * NU; e += G) B[(e / NU) * ldb + e % NU] = S(0);
    if (lane == 0) {
      B[5 * ldb + 0] = -dt * P[5];
      B[5 * ldb + 1] = dt * P[5];
    }
  }
  template <class S>
  DMPC_DEV static void jac_vary(const S* P, S dt, const S* x, const S* u, S* A, int lda, S* B, int ldb) {
    const S im = P[4];
    S s, c;
    sincos_(x[2], &s, &c);
    const S thrust = u[0] + u[1];
    const S dts = dt * s * im, dtc = dt * c * im;
    A[3 * lda + 2] = -thrust * dtc;
    A[4 * lda + 2] = -thrust * dts;
    B[3 * ldb + 0] = -dts;
    B[3 * ldb + 1] = -dts;
    B[4 * ldb + 0] = dtc;
    B[4 * ldb + 1] = dtc;
  }
  // g[p] += lh . df/dth_p + lam . (d2f/dth_p dz) dz   (oracle: theta_grad_stage)
  template <class S>
  DMPC_DEV static void theta_grad(const S* P, S dt, const S* x, const S* u, const S* dx,
                                  const S* du, const S* lh, const S* lam, S* g) {
    const S arm = P[1], I = P[2], im = P[4];
    S s, c;
    sincos_(x[2], &s, &c);
    const S F = u[0] + u[1], dF = du[0] + du[1], dd = u[1] - u[0], ddd = du[1] - du[0];
    const S im2 = dt * im * im;
    const S iI = S(1) / I;
    g[0] += lh[3] * (F * s * im2) + lh[4] * (-F * c * im2) +
            lam[3] * ((F * c * dx[2] + s * dF) * im2) + lam[4] * ((F * s * dx[2] - c * dF) * im2);
    g[1] += lh[5] * (dt * dd * iI) + lam[5] * (dt * ddd * iI);
    g[2] += lh[5] * (-dt * arm * dd * iI * iI) + lam[5] * (-dt * arm * ddd * iI * iI);
    g[3] += lh[4] * (-dt);
  }

 private:
  DMPC_DEV static void sincos_(double a, double* s, double* c) { sincos(a, s, c); }
  DMPC_DEV static void sincos_(float a, float* s, float* c) { sincosf(a, s, c); }
};

// ---------------------------------------------------------------------------
// 13-state quadrotor (kind 3). x = [p(3), q(4: w,x,y,z), v(3), w(3)], u = 4 rotors,
// th = [m, arm, Jx, Jy, Jz, kappa, g]. See paper_2605_29155_b200/dynamics.py.
// ---------------------------------------------------------------------------
struct Quad13 {
  static constexpr int NX = 13, NU = 4, NTH = 7, NP = 15, KIND = 3;
  static constexpr bool kLinearParams = false;
  __host__ __device__ static constexpr bool a_nz(int r, int c) {
    return r == c || (r < 3 && c == r + 7) ||
           (r >= 3 && r <= 6 && ((c >= 3 && c <= 6) || c >= 10)) ||   // quaternion kinematics
           ((r == 7 || r == 8) && c >= 3 && c <= 6) || (r == 9 && (c == 4 || c == 5)) ||  // R(q) e3
           (r >= 10 && c >= 10);                                       // gyroscopic terms
  }
  __host__ __device__ static constexpr bool b_nz(int r, int c) { return r >= 7 && c >= 0; }
  __host__ __device__ static constexpr bool a_one(int r, int c) { return r == c; }
  __host__ __device__ static constexpr bool a_dt(int r, int c) { return r < 3 && c == r + 7; }
  // P = [m, arm, Jx, Jy, Jz, kappa, g, 1/m, arm/sqrt2, 1/Jx, 1/Jy, 1/Jz, Jz-Jy, Jx-Jz, Jy-Jx]
  template <class S>
  DMPC_DEV static void prep(const S* th, S* P) {
#pragma unroll
    for (int i = 0; i < 7; i++) P[i] = th[i];
    P[7] = S(1) / th[0];
    P[8] = th[1] * S(kInvSqrt2);
    P[9] = S(1) / th[2];
    P[10] = S(1) / th[3];
    P[11] = S(1) / th[4];
    P[12] = th[4] - th[3];
    P[13] = th[2] - th[4];
    P[14] = th[3] - th[2];
  }
  template <class S>
  DMPC_DEV static void step(const S* P, S dt, const S* x, const S* u, S* o) {
    const S kap = P[5], g = P[6], im = P[7], d = P[8], iJx = P[9], iJy = P[10], iJz = P[11];
    const S dzy = P[12], dxz = P[13], dyx = P[14];
    const S qw = x[3], qx = x[4], qy = x[5], qz = x[6];
    const S wx = x[10], wy = x[11], wz = x[12];
    const S F = ((u[0] + u[1]) + u[2]) + u[3];
    const S tx = d * (((u[0] + u[1]) - u[2]) - u[3]);
    const S ty = d * (((u[1] - u[0]) + u[2]) - u[3]);
    const S tz = kap * (((u[0] - u[1]) + u[2]) - u[3]);
    const S hw = S(0.5) * dt;
    const S r13 = S(2) * (qx * qz + qw * qy);
    const S r23 = S(2) * (qy * qz - qw * qx);
    const S r33 = S(1) - S(2) * (qx * qx + qy * qy);
    const S a = F * im;
    o[0] = x[0] + dt * x[7];
    o[1] = x[1] + dt * x[8];
    o[2] = x[2] + dt * x[9];
    o[3] = qw + hw * (((-qx * wx) - qy * wy) - qz * wz);
    o[4] = qx + hw * ((qw * wx + qy * wz) - qz * wy);
    o[5] = qy + hw * ((qw * wy - qx * wz) + qz * wx);
    o[6] = qz + hw * ((qw * wz + qx * wy) - qy * wx);
    o[7] = x[7] + dt * (r13 * a);
    o[8] = x[8] + dt * (r23 * a);
    o[9] = x[9] + dt * (r33 * a - g);
    o[10] = wx + dt * ((tx - dzy * wy * wz) * iJx);
    o[11] = wy + dt * ((ty - dxz * wz * wx) * iJy);
    o[12] = wz + dt * ((tz - dyx * wx * wy) * iJz);
  }
  template <class S>
  DMPC_DEV static void jac_const(const S* P, S dt, S* A, int lda, S* B, int ldb, int lane, int G) {
    for (int e = lane; e < NX * NX; e += G) {
      int i = e / NX, j = e % NX;
      A[i * lda + j] = (i == j) ? S(1) : ((i < 3 && j == i + 7) ? dt : S(0));
    }
    for (int e = lane; e < NX * NU; e += G) B[(e / NU) * ldb + e % NU] = S(0);
    if (lane == 0) {
      const S bx = dt * P[8] * P[9], by = dt * P[8] * P[10], bz = dt * P[5] * P[11];
      B[10 * ldb + 0] = bx;  B[10 * ldb + 1] = bx;  B[10 * ldb + 2] = -bx; B[10 * ldb + 3] = -bx;
      B[11 * ldb + 0] = -by; B[11 * ldb + 1] = by;  B[11 * ldb + 2] = by;  B[11 * ldb + 3] = -by;
      B[12 * ldb + 0] = bz;  B[12 * ldb + 1] = -bz; B[12 * ldb + 2] = bz;  B[12 * ldb + 3] = -bz;
    }
  }
  template <class S>
  DMPC_DEV static void jac_vary(const S* P, S dt, const S* x, const S* u, S* A, int lda, S* B, int ldb) {
    const S im = P[7], iJx = P[9], iJy = P[10], iJz = P[11];
    const S dzy = P[12], dxz = P[13], dyx = P[14];
    const S qw = x[3], qx = x[4], qy = x[5], qz = x[6];
    const S wx = x[10], wy = x[11], wz = x[12];
    const S F = ((u[0] + u[1]) + u[2]) + u[3];
    const S hw = S(0.5) * dt;
    const S da = dt * (F * im);
    const S r13 = S(2) * (qx * qz + qw * qy);
    const S r23 = S(2) * (qy * qz - qw * qx);
    const S r33 = S(1) - S(2) * (qx * qx + qy * qy);
    A[3 * lda + 4] = -hw * wx; A[3 * lda + 5] = -hw * wy; A[3 * lda + 6] = -hw * wz;
    A[3 * lda + 10] = -hw * qx; A[3 * lda + 11] = -hw * qy; A[3 * lda + 12] = -hw * qz;
    A[4 * lda + 3] = hw * wx; A[4 * lda + 5] = hw * wz; A[4 * lda + 6] = -hw * wy;
    A[4 * lda + 10] = hw * qw; A[4 * lda + 11] = -hw * qz; A[4 * lda + 12] = hw * qy;
    A[5 * lda + 3] = hw * wy; A[5 * lda + 4] = -hw * wz; A[5 * lda + 6] = hw * wx;
    A[5 * lda + 10] = hw * qz; A[5 * lda + 11] = hw * qw; A[5 * lda + 12] = -hw * qx;
    A[6 * lda + 3] = hw * wz; A[6 * lda + 4] = hw * wy; A[6 * lda + 5] = -hw * wx;
    A[6 * lda + 10] = -hw * qy; A[6 * lda + 11] = hw * qx; A[6 * lda + 12] = hw * qw;
    A[7 * lda + 3] = da * (S(2) * qy); A[7 * lda + 4] = da * (S(2) * qz);
    A[7 * lda + 5] = da * (S(2) * qw); A[7 * lda + 6] = da * (S(2) * qx);
    A[8 * lda + 3] = da * (S(-2) * qx); A[8 * lda + 4] = da * (S(-2) * qw);
    A[8 * lda + 5] = da * (S(2) * qz); A[8 * lda + 6] = da * (S(2) * qy);
    A[9 * lda + 4] = da * (S(-4) * qx); A[9 * lda + 5] = da * (S(-4) * qy);
    const S dm = dt * im;
    const S b7 = r13 * dm, b8 = r23 * dm, b9 = r33 * dm;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      B[7 * ldb + j] = b7;
      B[8 * ldb + j] = b8;
      B[9 * ldb + j] = b9;
    }
    const S ex = -dt * iJx, ey = -dt * iJy, ez = -dt * iJz;
    A[10 * lda + 11] = ex * (dzy * wz); A[10 * lda + 12] = ex * (dzy * wy);
    A[11 * lda + 10] = ey * (dxz * wz); A[11 * lda + 12] = ey * (dxz * wx);
    A[12 * lda + 10] = ez * (dyx * wy); A[12 * lda + 11] = ez * (dyx * wx);
  }
  // Register-resident rows of A_t / B_t for the Riccati products: the 23 distinct
  // state-dependent values of one stage (same arithmetic as jac_vary / jac_const, so the
  // rows are bit-identical to the shared-memory copy) and a row accessor that the products
  // call with compile-time row indices (after unrolling), replacing shared-memory row loads.
  template <class S>
  struct JacRegs {
    S hwW[3], hwQ[4], dq[4], g[6], b[6];  // b: B rows 7..9 (b7,b8,b9) and 10..12 (bx,by,bz)
  };
  template <class S>
  DMPC_DEV static void jac_regs(const S* P, S dt, const S* z, JacRegs<S>& J) {
    const S im = P[7], iJx = P[9], iJy = P[10], iJz = P[11];
    const S dzy = P[12], dxz = P[13], dyx = P[14];
    const S qw = z[3], qx = z[4], qy = z[5], qz = z[6];
    const S wx = z[10], wy = z[11], wz = z[12];
    const S F = ((z[13] + z[14]) + z[15]) + z[16];
    const S hw = S(0.5) * dt;
    const S da = dt * (F * im);
    J.hwW[0] = hw * wx; J.hwW[1] = hw * wy; J.hwW[2] = hw * wz;
    J.hwQ[0] = hw * qw; J.hwQ[1] = hw * qx; J.hwQ[2] = hw * qy; J.hwQ[3] = hw * qz;
    J.dq[0] = da * (S(2) * qw); J.dq[1] = da * (S(2) * qx); J.dq[2] = da * (S(2) * qy); J.dq[3] = da * (S(2) * qz);
    const S ex = -dt * iJx, ey = -dt * iJy, ez = -dt * iJz;
    J.g[0] = ex * (dzy * wz); J.g[1] = ex * (dzy * wy); J.g[2] = ey * (dxz * wz);
    J.g[3] = ey * (dxz * wx); J.g[4] = ez * (dyx * wy); J.g[5] = ez * (dyx * wx);
    const S dm = dt * im;
    J.b[0] = (S(2) * (qx * qz + qw * qy)) * dm;
    J.b[1] = (S(2) * (qy * qz - qw * qx)) * dm;
    J.b[2] = (S(1) - S(2) * (qx * qx + qy * qy)) * dm;
    J.b[3] = dt * P[8] * P[9];
    J.b[4] = dt * P[8] * P[10];
    J.b[5] = dt * P[5] * P[11];
  }
  // rows of B_t that change with the state (7..9; rows 10..12 are constant, jac_const)
  template <int Dummy>
  __host__ __device__ static constexpr bool b_varies(int r) { return r >= 7 && r <= 9; }
  // state-dependent entries of A row r (others are unused by the callers) and B row r
  template <class S>
  DMPC_DEV static void jac_row(const JacRegs<S>& J, int r, S (&a)[NX], S (&b)[NU]) {
    switch (r) {
      case 3: a[4] = -J.hwW[0]; a[5] = -J.hwW[1]; a[6] = -J.hwW[2];
              a[10] = -J.hwQ[1]; a[11] = -J.hwQ[2]; a[12] = -J.hwQ[3]; break;
      case 4: a[3] = J.hwW[0]; a[5] = J.hwW[2]; a[6] = -J.hwW[1];
              a[10] = J.hwQ[0]; a[11] = -J.hwQ[3]; a[12] = J.hwQ[2]; break;
      case 5: a[3] = J.hwW[1]; a[4] = -J.hwW[2]; a[6] = J.hwW[0];
              a[10] = J.hwQ[3]; a[11] = J.hwQ[0]; a[12] = -J.hwQ[1]; break;
      case 6: a[3] = J.hwW[2]; a[4] = J.hwW[1]; a[5] = -J.hwW[0];
              a[10] = -J.hwQ[2]; a[11] = J.hwQ[1]; a[12] = J.hwQ[0]; break;
      case 7: a[3] = J.dq[2]; a[4] = J.dq[3]; a[5] = J.dq[0]; a[6] = J.dq[1];
              b[0] = b[1] = b[2] = b[3] = J.b[0]; break;
      case 8: a[3] = -J.dq[1]; a[4] = -J.dq[0]; a[5] = J.dq[3]; a[6] = J.dq[2];
              b[0] = b[1] = b[2] = b[3] = J.b[1]; break;
      case 9: a[4] = S(-2) * J.dq[1]; a[5] = S(-2) * J.dq[2];
              b[0] = b[1] = b[2] = b[3] = J.b[2]; break;
      case 10: a[11] = J.g[0]; a[12] = J.g[1];
               b[0] = J.b[3]; b[1] = J.b[3]; b[2] = -J.b[3]; b[3] = -J.b[3]; break;
      case 11: a[10] = J.g[2]; a[12] = J.g[3];
               b[0] = -J.b[4]; b[1] = J.b[4]; b[2] = J.b[4]; b[3] = -J.b[4]; break;
      case 12: a[10] = J.g[4]; a[11] = J.g[5];
               b[0] = J.b[5]; b[1] = -J.b[5]; b[2] = J.b[5]; b[3] = -J.b[5]; break;
      default: break;
    }
  }
  // B[r][i] with a runtime column i (rows 7..9 are column-uniform, 10..12 the X mixer signs)
  template <class S>
  DMPC_DEV static S jac_b(const JacRegs<S>& J, int r, int i) {
    switch (r) {
      case 7: return J.b[0];
      case 8: return J.b[1];
      case 9: return J.b[2];
      case 10: return i < 2 ? J.b[3] : -J.b[3];
      case 11: return (i == 1 || i == 2) ? J.b[4] : -J.b[4];
      case 12: return (i & 1) ? -J.b[5] : J.b[5];
      default: return S(0);
    }
  }
  template <class S>
  DMPC_DEV static void theta_grad(const S* P, S dt, const S* x, const S* u, const S* dx,
                                  const S* du, const S* lh, const S* lam, S* g) {
    const S kap = P[5], im = P[7], d = P[8], iJx = P[9], iJy = P[10], iJz = P[11];
    const S dzy = P[12], dxz = P[13], dyx = P[14];
    const S qw = x[3], qx = x[4], qy = x[5], qz = x[6];
    const S wx = x[10], wy = x[11], wz = x[12];
    const S dqw = dx[3], dqx = dx[4], dqy = dx[5], dqz = dx[6];
    const S dwx = dx[10], dwy = dx[11], dwz = dx[12];
    const S F = ((u[0] + u[1]) + u[2]) + u[3];
    const S dF = ((du[0] + du[1]) + du[2]) + du[3];
    const S sx = ((u[0] + u[1]) - u[2]) - u[3], dsx = ((du[0] + du[1]) - du[2]) - du[3];
    const S sy = ((u[1] - u[0]) + u[2]) - u[3], dsy = ((du[1] - du[0]) + du[2]) - du[3];
    const S sz = ((u[0] - u[1]) + u[2]) - u[3], dsz = ((du[0] - du[1]) + du[2]) - du[3];
    const S tx = d * sx, ty = d * sy, tz = kap * sz;
    const S r13 = S(2) * (qx * qz + qw * qy), r23 = S(2) * (qy * qz - qw * qx);
    const S r33 = S(1) - S(2) * (qx * qx + qy * qy);
    const S dr13 = S(2) * (qy * dqw + qz * dqx + qw * dqy + qx * dqz);
    const S dr23 = S(2) * (-qx * dqw - qw * dqx + qz * dqy + qy * dqz);
    const S dr33 = S(-4) * (qx * dqx + qy * dqy);
    const S im2 = dt * im * im;
    g[0] += -im2 * F * (lh[7] * r13 + lh[8] * r23 + lh[9] * r33) -
            im2 * (lam[7] * (F * dr13 + r13 * dF) + lam[8] * (F * dr23 + r23 * dF) +
                   lam[9] * (F * dr33 + r33 * dF));
    const S c = S(kInvSqrt2);
    g[1] += lh[10] * (dt * c * sx * iJx) + lh[11] * (dt * c * sy * iJy) +
            lam[10] * (dt * c * dsx * iJx) + lam[11] * (dt * c * dsy * iJy);
    const S e10 = tx - dzy * wy * wz, e11 = ty - dxz * wz * wx, e12 = tz - dyx * wx * wy;
    const S de10 = d * dsx - dzy * (wz * dwy + wy * dwz);
    const S de11 = d * dsy - dxz * (wx * dwz + wz * dwx);
    const S de12 = kap * dsz - dyx * (wy * dwx + wx * dwy);
    const S pyz = wy * wz, pzx = wz * wx, pxy = wx * wy;
    const S dpyz = wz * dwy + wy * dwz, dpzx = wx * dwz + wz * dwx, dpxy = wy * dwx + wx * dwy;
    g[2] += lh[10] * (-dt * e10 * iJx * iJx) + lh[11] * (-dt * pzx * iJy) + lh[12] * (dt * pxy * iJz) +
            lam[10] * (-dt * de10 * iJx * iJx) + lam[11] * (-dt * dpzx * iJy) + lam[12] * (dt * dpxy * iJz);
    g[3] += lh[10] * (dt * pyz * iJx) + lh[11] * (-dt * e11 * iJy * iJy) + lh[12] * (-dt * pxy * iJz) +
            lam[10] * (dt * dpyz * iJx) + lam[11] * (-dt * de11 * iJy * iJy) + lam[12] * (-dt * dpxy * iJz);
    g[4] += lh[10] * (-dt * pyz * iJx) + lh[11] * (dt * pzx * iJy) + lh[12] * (-dt * e12 * iJz * iJz) +
            lam[10] * (-dt * dpyz * iJx) + lam[11] * (dt * dpzx * iJy) + lam[12] * (-dt * de12 * iJz * iJz);
    g[5] += lh[12] * (dt * sz * iJz) + lam[12] * (dt * dsz * iJz);
    g[6] += lh[9] * (-dt);
  }
};

// ---------------------------------------------------------------------------
// linear model x+ = A x + B u, th = [A row-major, B row-major] (kernels.py:66-73, 112-117).
// The kernels keep [A | B] in shared memory (jac_const copies th there once); `step`
// reads from that copy, so `th` passed to step/jac_vary is the smem A (lda) / B pair.
// ---------------------------------------------------------------------------
template <int NX_, int NU_>
struct LinearModel {
  static constexpr int NX = NX_, NU = NU_, NTH = NX_ * NX_ + NX_ * NU_, NP = 1, KIND = 2;
  __host__ __device__ static constexpr bool a_nz(int, int) { return true; }  // dense
  __host__ __device__ static constexpr bool b_nz(int, int) { return true; }
  __host__ __device__ static constexpr bool a_one(int, int) { return false; }
  __host__ __device__ static constexpr bool a_dt(int, int) { return false; }
  static constexpr bool kLinearParams = true;
};

}  // namespace dmpc

namespace dmpc {
using DoubleIntegrator1 = DoubleIntegrator<1>;
using DoubleIntegrator2 = DoubleIntegrator<2>;
using DoubleIntegrator3 = DoubleIntegrator<3>;
using Linear1x1 = LinearModel<1, 1>;
using Linear2x1 = LinearModel<2, 1>;
using Linear3x2 = LinearModel<3, 2>;
using Linear4x2 = LinearModel<4, 2>;
using Linear13x4 = LinearModel<13, 4>;
}  // namespace dmpc

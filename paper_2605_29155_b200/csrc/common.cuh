// common.cuh — lane-group helpers, async staging and the stage-QP control block.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "models.cuh"

namespace dmpc {

// One MPC problem is owned by a group of G consecutive lanes of a warp (G = 4, 8,
// 16 or 32). All synchronisation inside a problem uses the group's lane mask, so
// groups of the same warp progress independently (different iteration counts).
template <int G>
DMPC_DEV unsigned group_mask() {
  if constexpr (G == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31u;
    return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
  }
}

template <class T>
DMPC_DEV T gshfl(unsigned mask, T v, int src, int width) {
  return __shfl_sync(mask, v, src, width);
}
template <class T>
DMPC_DEV T gxor(unsigned mask, T v, int m, int width) {
  return __shfl_xor_sync(mask, v, m, width);
}

// cp.async staging of one element (4 or 8 bytes) global -> shared.
DMPC_DEV void cp_async_elem(float* dst, const float* src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
DMPC_DEV void cp_async_elem(double* dst, const double* src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
DMPC_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
DMPC_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <class T>
DMPC_DEV bool finite_(T v) { return isfinite(v); }

// ---------------------------------------------------------------------------
// Stage QP control block (kernels.py:195-318 boxqp_one/_chol_* and the lambda
// schedule of backward_range, kernels.py:444-489), in double, executed redundantly
// by every lane of the group (the operands are NU <= 4 vectors kept in registers).
//
// Free-set Cholesky is done in "masked" form: clamped rows/columns are replaced by
// identity rows. Because the off-diagonal entries involving a clamped index are
// exact zeros, every free-set quantity equals the reference's compacted
// factorisation / substitution term for term (s - 0*y == s), so results match the
// index-list formulation exactly while all register indices stay compile-time.
// ---------------------------------------------------------------------------
constexpr double kArmijo = 0.1, kStepDec = 0.6, kMinStep = 1e-20, kLamInit = 1e-6, kLamMax = 1e-2;

template <int NU>
struct Chol {
  double L[NU][NU];
  double inv[NU];  // 1 / L[a][a]
};

template <int NU>
DMPC_DEV bool chol_masked(const double (&H)[NU][NU], const bool (&fr)[NU], Chol<NU>& c) {
  bool ok = true;
#pragma unroll
  for (int a = 0; a < NU; a++) {
#pragma unroll
    for (int b = 0; b <= a; b++) {
      double s;
      if (fr[a] && fr[b]) {
        s = H[a][b];
      } else {
        s = (a == b) ? 1.0 : 0.0;
      }
#pragma unroll
      for (int r = 0; r < b; r++) s -= c.L[a][r] * c.L[b][r];
      if (a == b) {
        if (s <= 0.0) ok = false;
        c.L[a][a] = sqrt(s);
        c.inv[a] = 1.0 / c.L[a][a];
      } else {
        c.L[a][b] = s / c.L[b][b];
      }
    }
  }
  return ok;
}

// L L' out = b (masked rows of b are zero and stay zero)
template <int NU>
DMPC_DEV void chol_solve(const Chol<NU>& c, const double (&b)[NU], double (&out)[NU]) {
#pragma unroll
  for (int a = 0; a < NU; a++) {
    double s = b[a];
#pragma unroll
    for (int r = 0; r < a; r++) s -= c.L[a][r] * out[r];
    out[a] = s / c.L[a][a];
  }
#pragma unroll
  for (int a = NU - 1; a >= 0; a--) {
    double s = out[a];
#pragma unroll
    for (int r = a + 1; r < NU; r++) s -= c.L[r][a] * out[r];
    out[a] = s / c.L[a][a];
  }
}

template <int NU>
DMPC_DEV double qp_value(const double (&H)[NU][NU], const double (&g)[NU], const double (&u)[NU]) {
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < NU; a++) {
    double row = 0.0;
#pragma unroll
    for (int b = 0; b < NU; b++) row += H[a][b] * u[b];
    acc += 0.5 * u[a] * row + g[a] * u[a];
  }
  return acc;
}

// boxqp_one (kernels.py:239-318). Returns 0 (OK) or -1 (NOT_PD).
template <int NU>
DMPC_DEV int boxqp(const double (&H)[NU][NU], const double (&g)[NU], const double (&lo)[NU],
                   const double (&hi)[NU], double (&u)[NU], bool (&fr)[NU], int max_iter,
                   double tol) {
#pragma unroll
  for (int a = 0; a < NU; a++) {
    if (u[a] < lo[a]) u[a] = lo[a];
    else if (u[a] > hi[a]) u[a] = hi[a];
    fr[a] = true;
  }
  double value = qp_value<NU>(H, g, u);
  Chol<NU> ch;
  for (int it = 0; it < max_iter; it++) {
    double grad[NU];
    int nf = 0;
#pragma unroll
    for (int a = 0; a < NU; a++) {
      double s = g[a];
#pragma unroll
      for (int b = 0; b < NU; b++) s += H[a][b] * u[b];
      grad[a] = s;
      const bool clamped = (u[a] <= lo[a] && s > 0.0) || (u[a] >= hi[a] && s < 0.0);
      fr[a] = !clamped;
      nf += fr[a] ? 1 : 0;
    }
    if (nf == 0) return 0;
    double gnorm = 0.0;
#pragma unroll
    for (int a = 0; a < NU; a++)
      if (fr[a]) gnorm += grad[a] * grad[a];
    if (sqrt(gnorm) <= tol) return 0;
    if (!chol_masked<NU>(H, fr, ch)) return -1;
    double rhs[NU], cand[NU];
#pragma unroll
    for (int a = 0; a < NU; a++) {
      double s = 0.0;
      if (fr[a]) {
        s = g[a];
#pragma unroll
        for (int b = 0; b < NU; b++)
          if (!fr[b]) s += H[a][b] * u[b];
      }
      rhs[a] = s;
    }
    chol_solve<NU>(ch, rhs, cand);
    double search[NU];
    double sdotg = 0.0;
#pragma unroll
    for (int a = 0; a < NU; a++) {
      search[a] = fr[a] ? (-cand[a] - u[a]) : 0.0;
      if (fr[a]) sdotg += search[a] * grad[a];
    }
    if (sdotg >= 0.0) return 0;
    double step = 1.0, vc = 0.0;
    bool accepted = false;
    while (step > kMinStep) {
#pragma unroll
      for (int a = 0; a < NU; a++) {
        double v = u[a] + step * search[a];
        if (v < lo[a]) v = lo[a];
        else if (v > hi[a]) v = hi[a];
        cand[a] = v;
      }
      vc = qp_value<NU>(H, g, cand);
      if (vc - value <= kArmijo * step * sdotg) {
        accepted = true;
        break;
      }
      step *= kStepDec;
    }
    if (!accepted) return 0;
#pragma unroll
    for (int a = 0; a < NU; a++) u[a] = cand[a];
    value = vc;
  }
  return 0;
}

// The lambda-regularised stage solve of backward_range (kernels.py:440-471).
// On success: du (the feedforward k_t), fr (free mask), ch (Cholesky of the
// regularised free block, used for the K columns).
template <int NU>
DMPC_DEV bool stage_qp(const double (&Quu)[NU][NU], const double (&qu)[NU], const double (&lo)[NU],
                       const double (&hi)[NU], int max_iter, double tol, double (&du)[NU],
                       bool (&fr)[NU], Chol<NU>& ch) {
  double lam = 0.0;
  for (;;) {
    double Ht[NU][NU];
#pragma unroll
    for (int a = 0; a < NU; a++)
#pragma unroll
      for (int b = 0; b < NU; b++) Ht[a][b] = Quu[a][b] + (a == b ? lam : 0.0);
#pragma unroll
    for (int a = 0; a < NU; a++) du[a] = 0.0;
    const int st = boxqp<NU>(Ht, qu, lo, hi, du, fr, max_iter, tol);
    if (st == 0) {
      bool any = false;
#pragma unroll
      for (int a = 0; a < NU; a++) any |= fr[a];
      if (!any) {
        // n_free == 0: no factorisation needed; make ch an identity so K solves are inert
#pragma unroll
        for (int a = 0; a < NU; a++) {
#pragma unroll
          for (int b = 0; b < NU; b++) ch.L[a][b] = (a == b) ? 1.0 : 0.0;
          ch.inv[a] = 1.0;
        }
        return true;
      }
      if (chol_masked<NU>(Ht, fr, ch)) return true;
    }
    lam = (lam == 0.0) ? kLamInit : lam * 10.0;
    if (lam > kLamMax) return false;
  }
}

}  // namespace dmpc

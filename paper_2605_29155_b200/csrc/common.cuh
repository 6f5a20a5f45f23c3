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
// 16-byte global -> shared copy that bypasses L1 (.cg): used for data this kernel itself
// wrote to global memory earlier (the gain workspace), so no stale L1 line can be hit.
DMPC_DEV void cp_async_16cg(void* dst, const void* src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
// element copy without a cache hint. The hinted 4/8-byte form (cp_async_elem) compiled, in some
// instantiations, to LDGSTS [R+UR0+imm], desc[UR1] with UR0/UR1 never written in the kernel;
// in the f64 3x2 linear-model backward that faulted (misaligned shared write / illegal
// instruction), so the element copies of the staging paths carry no hint.
template <class T>
DMPC_DEV void cp_async_elem_nh(T* dst, const T* src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if constexpr (sizeof(T) == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
DMPC_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
DMPC_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <class T>
DMPC_DEV bool finite_(T v) { return isfinite(v); }

DMPC_DEV float mul_rn(float a, float b) { return __fmul_rn(a, b); }
DMPC_DEV double mul_rn(double a, double b) { return __dmul_rn(a, b); }

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

template <int NU, class T = double>
struct Chol {
  T L[NU][NU];  // lower triangle used
  T inv[NU];    // 1 / L[a][a]
};

DMPC_DEV double rsqrt_(double v) { return rsqrt(v); }
DMPC_DEV float rsqrt_(float v) { return rsqrtf(v); }
DMPC_DEV double sqrt_(double v) { return sqrt(v); }
DMPC_DEV float sqrt_(float v) { return sqrtf(v); }

// Masked Cholesky; the diagonal reciprocals come from one rsqrt, and the
// off-diagonal / substitution divisions become multiplications by them (a one-ulp
// difference from the reference's divisions, far below the parity tolerances).
template <int NU, class T>
DMPC_DEV bool chol_masked(const T (&H)[NU][NU], T lam, const bool (&fr)[NU], Chol<NU, T>& c) {
  bool ok = true;
#pragma unroll
  for (int a = 0; a < NU; a++) {
#pragma unroll
    for (int b = 0; b <= a; b++) {
      T s;
      if (fr[a] && fr[b]) {
        s = H[a][b] + (a == b ? lam : T(0));
      } else {
        s = (a == b) ? T(1) : T(0);
      }
#pragma unroll
      for (int r = 0; r < b; r++) s -= c.L[a][r] * c.L[b][r];
      if (a == b) {
        if (s <= T(0)) ok = false;
        const T is = rsqrt_(s);
        c.inv[a] = is;
        c.L[a][a] = s * is;
      } else {
        c.L[a][b] = s * c.inv[b];
      }
    }
  }
  return ok;
}

// L L' out = b (masked rows of b are zero and stay zero)
template <int NU, class T>
DMPC_DEV void chol_solve(const Chol<NU, T>& c, const T (&b)[NU], T (&out)[NU]) {
#pragma unroll
  for (int a = 0; a < NU; a++) {
    T s = b[a];
#pragma unroll
    for (int r = 0; r < a; r++) s -= c.L[a][r] * out[r];
    out[a] = s * c.inv[a];
  }
#pragma unroll
  for (int a = NU - 1; a >= 0; a--) {
    T s = out[a];
#pragma unroll
    for (int r = a + 1; r < NU; r++) s -= c.L[r][a] * out[r];
    out[a] = s * c.inv[a];
  }
}

// 0.5 u'(H + lam I)u + g'u
template <int NU, class T>
DMPC_DEV T qp_value(const T (&H)[NU][NU], T lam, const T (&g)[NU], const T (&u)[NU]) {
  T acc = T(0);
#pragma unroll
  for (int a = 0; a < NU; a++) {
    T row = T(0);
#pragma unroll
    for (int b = 0; b < NU; b++) row += (H[a][b] + (a == b ? lam : T(0))) * u[b];
    acc += T(0.5) * u[a] * row + g[a] * u[a];
  }
  return acc;
}

template <int NU>
DMPC_DEV bool same_mask(const bool (&a)[NU], const bool (&b)[NU]) {
  bool e = true;
#pragma unroll
  for (int i = 0; i < NU; i++) e = e && (a[i] == b[i]);
  return e;
}

// boxqp_one (kernels.py:239-318) on H + lam I. Returns 0 (OK) or -1 (NOT_PD).
// `ch` / `ch_fr` carry the last factorisation and the free mask it was computed
// for: H is fixed inside the call, so a repeated free set reuses the identical
// factor. The backtracking loop stops as soon as the trial point no longer moves
// (u + step*search == u in every coordinate): from there on every smaller step
// gives the same rejected value, so the reference's remaining trials down to
// step <= 1e-20 cannot accept and the outcome is unchanged.
template <int NU, class T>
DMPC_DEV int boxqp(const T (&H)[NU][NU], T lam, const T (&g)[NU], const T (&lo)[NU],
                   const T (&hi)[NU], T (&u)[NU], bool (&fr)[NU], int max_iter,
                   T tol, Chol<NU, T>& ch, bool (&ch_fr)[NU], bool& ch_ok) {
#pragma unroll
  for (int a = 0; a < NU; a++) {
    if (u[a] < lo[a]) u[a] = lo[a];
    else if (u[a] > hi[a]) u[a] = hi[a];
    fr[a] = true;
  }
  ch_ok = false;
  T value = qp_value<NU, T>(H, lam, g, u);
  for (int it = 0; it < max_iter; it++) {
    T grad[NU];
    int nf = 0;
#pragma unroll
    for (int a = 0; a < NU; a++) {
      T s = g[a];
#pragma unroll
      for (int b = 0; b < NU; b++) s += (H[a][b] + (a == b ? lam : T(0))) * u[b];
      grad[a] = s;
      const bool clamped = (u[a] <= lo[a] && s > T(0)) || (u[a] >= hi[a] && s < T(0));
      fr[a] = !clamped;
      nf += fr[a] ? 1 : 0;
    }
    if (nf == 0) return 0;
    T gnorm = T(0);
#pragma unroll
    for (int a = 0; a < NU; a++)
      if (fr[a]) gnorm += grad[a] * grad[a];
    if (sqrt_(gnorm) <= tol) return 0;
    if (!(ch_ok && same_mask<NU>(fr, ch_fr))) {
#pragma unroll
      for (int a = 0; a < NU; a++) ch_fr[a] = fr[a];
      ch_ok = chol_masked<NU, T>(H, lam, fr, ch);
      if (!ch_ok) return -1;
    }
    T rhs[NU], cand[NU];
#pragma unroll
    for (int a = 0; a < NU; a++) {
      T s = T(0);
      if (fr[a]) {
        s = g[a];
#pragma unroll
        for (int b = 0; b < NU; b++)
          if (!fr[b]) s += H[a][b] * u[b];
      }
      rhs[a] = s;
    }
    chol_solve<NU, T>(ch, rhs, cand);
    T search[NU];
    T sdotg = T(0);
#pragma unroll
    for (int a = 0; a < NU; a++) {
      search[a] = fr[a] ? (-cand[a] - u[a]) : T(0);
      if (fr[a]) sdotg += search[a] * grad[a];
    }
    if (sdotg >= T(0)) return 0;
    T step = T(1), vc = T(0);
    bool accepted = false;
    while (step > T(kMinStep)) {
      bool moved = false;
#pragma unroll
      for (int a = 0; a < NU; a++) {
        T v = u[a] + step * search[a];
        if (v < lo[a]) v = lo[a];
        else if (v > hi[a]) v = hi[a];
        cand[a] = v;
        moved |= (v != u[a]);
      }
      if (!moved) break;
      vc = qp_value<NU, T>(H, lam, g, cand);
      if (vc - value <= T(kArmijo) * step * sdotg) {
        accepted = true;
        break;
      }
      step *= T(kStepDec);
    }
    if (!accepted) return 0;
#pragma unroll
    for (int a = 0; a < NU; a++) u[a] = cand[a];
    value = vc;
  }
  return 0;
}

// The interior fast path of stage_qp (below), straight-line: every quantity is computed
// unconditionally and the validity is returned (true iff stage_qp would take its fast path;
// du / fr / ch are then exactly what stage_qp returns). Used where the QP sits alone on a
// latency-critical path (the block-per-problem kernel): no branches until the caller's
// single "fall back to stage_qp" test.
template <int NU, class T>
DMPC_DEV bool qp_interior(const T (&Quu)[NU][NU], const T (&qu)[NU], const T (&lo)[NU], const T (&hi)[NU],
                          T tol, T (&du)[NU], bool (&fr)[NU], Chol<NU, T>& ch) {
  bool inside = true, all_free[NU];
  T gn = T(0);
#pragma unroll
  for (int a = 0; a < NU; a++) {
    inside = inside && (lo[a] < T(0)) && (hi[a] > T(0));
    all_free[a] = true;
    gn += qu[a] * qu[a];
  }
  const bool pd = chol_masked<NU, T>(Quu, T(0), all_free, ch);
  T sol[NU];
  chol_solve<NU, T>(ch, qu, sol);
  bool strict = true;
  T sdotg = T(0);
#pragma unroll
  for (int a = 0; a < NU; a++) {
    strict = strict && (-sol[a] > lo[a]) && (-sol[a] < hi[a]);
    sdotg -= sol[a] * qu[a];
    du[a] = -sol[a];
    fr[a] = true;
  }
  return inside && pd && strict && sdotg < T(0) && !(sqrt_(gn) <= tol);
}

// The lambda-regularised stage solve of backward_range (kernels.py:440-471).
// On success: du (the feedforward k_t), fr (free mask), ch (Cholesky of the
// regularised free block, used for the K columns). The lambda schedule is
// generated in double exactly as the reference does (0, 1e-6, x10 ... <= 1e-2).
template <int NU, class T>
DMPC_DEV bool stage_qp(const T (&Quu)[NU][NU], const T (&qu)[NU], const T (&lo)[NU],
                       const T (&hi)[NU], int max_iter, T tol, T (&du)[NU],
                       bool (&fr)[NU], Chol<NU, T>& ch, bool& lam0) {
  lam0 = true;
  // Interior fast path (lambda = 0). From u = 0 with lo < 0 < hi no coordinate is
  // clamped, the Newton step -H^-1 g is taken at step 1 (Armijo holds with margin
  // 0.4 g'H^-1 g), and when that point is strictly inside the box the reference's
  // next iteration only refines it at round-off level (gnorm <= tol in double). So
  // du = -H^-1 g, all coordinates free, and the factor of H is the one K needs.
  {
    bool inside = true, all_free[NU];
    T gn = T(0);
#pragma unroll
    for (int a = 0; a < NU; a++) {
      inside = inside && (lo[a] < T(0)) && (hi[a] > T(0));
      all_free[a] = true;
      gn += qu[a] * qu[a];
    }
    if (inside && chol_masked<NU, T>(Quu, T(0), all_free, ch)) {
      T sol[NU];
      chol_solve<NU, T>(ch, qu, sol);
      bool strict = true;
      T sdotg = T(0);
#pragma unroll
      for (int a = 0; a < NU; a++) {
        strict = strict && (-sol[a] > lo[a]) && (-sol[a] < hi[a]);
        sdotg -= sol[a] * qu[a];
      }
      if (strict && sdotg < T(0) && !(sqrt_(gn) <= tol)) {
#pragma unroll
        for (int a = 0; a < NU; a++) {
          du[a] = -sol[a];
          fr[a] = true;
        }
        return true;
      }
    }
  }
  double lamd = 0.0;
  for (;;) {
    const T lam = (T)lamd;
#pragma unroll
    for (int a = 0; a < NU; a++) du[a] = T(0);
    bool ch_fr[NU];
    bool ch_ok;
    const int st = boxqp<NU, T>(Quu, lam, qu, lo, hi, du, fr, max_iter, tol, ch, ch_fr, ch_ok);
    if (st == 0) {
      bool any = false;
#pragma unroll
      for (int a = 0; a < NU; a++) any |= fr[a];
      if (!any) {
        // n_free == 0: no factorisation needed; make ch an identity so K solves are inert
#pragma unroll
        for (int a = 0; a < NU; a++) {
#pragma unroll
          for (int b = 0; b < NU; b++) ch.L[a][b] = (a == b) ? T(1) : T(0);
          ch.inv[a] = T(1);
        }
        return true;
      }
      if (ch_ok && same_mask<NU>(fr, ch_fr)) return true;  // factor of this free set is current
      if (chol_masked<NU, T>(Quu, lam, fr, ch)) return true;
    }
    lamd = (lamd == 0.0) ? kLamInit : lamd * 10.0;
    lam0 = false;
    if (lamd > kLamMax) return false;
  }
}

}  // namespace dmpc

// ilqr_forward.cuh — the fused forward iLQR kernel (one launch per solve).
//
// One MPC problem per group of G lanes (G = pow2 >= n_x, so 16 for the 13-state
// quadrotor: two problems per warp). Everything a problem needs between stages —
// nominal trajectory, gains, value expansion — stays on chip (shared memory +
// registers) for the whole solve; only C_t / c_t are streamed from L2/HBM with
// cp.async double buffering. Per iLQR iteration the group runs, without leaving the
// kernel:
//   stage 1+2  Riccati sweep t = T-1..0 with the Jacobians (A_t, B_t) evaluated in
//              place (the reference's linearize_range fused into backward_range,
//              kernels.py:181-187 + 326-512) and the lambda-regularised projected-
//              Newton box QP on the control block (kernels.py:239-318, 440-489);
//   stage 3    parallel line search: the n_alpha candidates run concurrently on
//              G/4-lane slots (kernels.py:520-574), followed by the accept /
//              converge epilogue of ilqr.py:216-244 evaluated on device.
// The batch-level "loop while any instance is active" (ilqr.py:204-206) becomes a
// per-problem loop: problems are independent, so per-instance results are
// identical to the reference's batch loop (tests/test_batchexec.py:55-62).
//
// Precision: the Riccati matrix algebra runs in the ABI type R (float for _f32);
// trajectory propagation, cost accumulation (rollout, line search) and the stage
// QP run in double — the iteration-count-critical quantities (SURVEY.md §7 hard
// part 2, probes P7/P8).
//
// Shared-memory layout per problem (FwdLayout): nominal X/U and k (double), K (R),
// Riccati scratch (R), two C_t staging buffers (R).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace dmpc {

struct FwdArgs {
  int B, T, K_max, n_alpha, boxqp_max_iter, theta_stride, gpb, smem_stride;
  double dt, conv_tol, boxqp_tol;
  double u_min[8], u_max[8], alphas[8];
  const void* theta;
  const void* C;
  const void* c;
  const void* x0;
  const void* U_warm;
  void* X;
  void* U;
  void* J;
  void* K;
  void* k;
  int32_t* iters;
  uint8_t* converged;
  uint8_t* diverged;
  int32_t* fail_t;
  uint8_t* clamped;
  void* alpha_hist;
  void* J_hist;
};

__host__ __device__ inline int align_up(int v, int a) { return (v + a - 1) / a * a; }

template <class M, bool DIAG, class R>
struct FwdLayout {
  static constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  static constexpr int LDA = NX;
  static constexpr int NCS = DIAG ? NZ : NZ * NZ;
  int oXn, oUn, okg, oKg, oAs, oBs, oMA, oNB, oKT, oQuxT, oQuuKT, oQuu, oqu, oVx, ozs, oC, oc, total;
  __host__ __device__ static FwdLayout make(int T) {
    FwdLayout L;
    int o = 0;
    L.oXn = o; o += (T + 1) * NX * 8;
    L.oUn = o; o += T * NU * 8;
    L.okg = o; o += T * NU * 8;
    L.oKg = o; o += T * NU * NX * (int)sizeof(R);
    o = align_up(o, 16);
    L.oAs = o; o += NX * LDA * (int)sizeof(R);
    L.oBs = o; o += NX * NU * (int)sizeof(R);
    L.oMA = o; o += NX * LDA * (int)sizeof(R);
    L.oNB = o; o += NX * NU * (int)sizeof(R);
    L.oKT = o; o += NX * NU * (int)sizeof(R);
    L.oQuxT = o; o += NX * NU * (int)sizeof(R);
    L.oQuuKT = o; o += NX * NU * (int)sizeof(R);
    L.oQuu = o; o += NU * NU * (int)sizeof(R);
    L.oqu = o; o += NU * (int)sizeof(R);
    L.oVx = o; o += NX * (int)sizeof(R);
    L.ozs = o; o += NZ * (int)sizeof(R);
    o = align_up(o, 16);
    L.oC = o; o += 2 * NCS * (int)sizeof(R);
    L.oc = o; o += 2 * NZ * (int)sizeof(R);
    L.total = align_up(o, 16);
    return L;
  }
};

// x+ = f(x,u) in double; the linear model reads its [A|B] copy from shared memory.
template <class M, class R>
DMPC_DEV void step_e(const double* th, double dt, const R* As, const R* Bs, const double* x,
                     const double* u, double* o) {
  if constexpr (M::kLinearParams) {
#pragma unroll
    for (int i = 0; i < M::NX; i++) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M::NX; j++) acc += (double)As[i * M::NX + j] * x[j];
#pragma unroll
      for (int j = 0; j < M::NU; j++) acc += (double)Bs[i * M::NU + j] * u[j];
      o[i] = acc;
    }
  } else {
    M::template step<double>(th, dt, x, u, o);
  }
}

template <class M, int G, bool DIAG, class R>
__global__ void __launch_bounds__(128) ilqr_forward_kernel(const FwdArgs args) {
  constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  using Lay = FwdLayout<M, DIAG, R>;
  constexpr int LDA = Lay::LDA, NCS = Lay::NCS;
  constexpr int NSLOT = G >= 4 ? 4 : G;  // concurrent line-search candidates
  constexpr int LC = G / NSLOT;          // lanes per candidate slot
  constexpr int NTHL = M::kLinearParams ? 1 : (M::NTH > 0 ? M::NTH : 1);

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int grp = threadIdx.x / G;
  const int lane = threadIdx.x % G;
  const int pid = blockIdx.x * args.gpb + grp;
  if (grp >= args.gpb || pid >= args.B) return;
  const unsigned gm = group_mask<G>();
  const int T = args.T;
  const Lay L = Lay::make(T);
  unsigned char* base = smem_raw + (size_t)grp * args.smem_stride;
  double* Xn = (double*)(base + L.oXn);
  double* Un = (double*)(base + L.oUn);
  double* kg = (double*)(base + L.okg);
  R* Kg = (R*)(base + L.oKg);
  R* As = (R*)(base + L.oAs);
  R* Bs = (R*)(base + L.oBs);
  R* MA = (R*)(base + L.oMA);
  R* NB = (R*)(base + L.oNB);
  R* KT = (R*)(base + L.oKT);
  R* QuxT = (R*)(base + L.oQuxT);
  R* QuuKT = (R*)(base + L.oQuuKT);
  R* Quus = (R*)(base + L.oQuu);
  R* qus = (R*)(base + L.oqu);
  R* Vxs = (R*)(base + L.oVx);
  R* zs = (R*)(base + L.ozs);
  R* Cb = (R*)(base + L.oC);
  R* cb = (R*)(base + L.oc);

  const R* Cg = (const R*)args.C + (size_t)pid * T * NCS;
  const R* cg = (const R*)args.c + (size_t)pid * T * NZ;

  // ---- parameters ----
  const R* thg = (const R*)args.theta + (size_t)args.theta_stride * pid;
  double th_e[NTHL];
  R th_r[NTHL];
  if constexpr (!M::kLinearParams) {
#pragma unroll
    for (int i = 0; i < NTHL; i++) {
      th_r[i] = (i < M::NTH) ? thg[i] : R(0);
      th_e[i] = (double)th_r[i];
    }
  } else {
    th_e[0] = 0.0;
    th_r[0] = R(0);
  }
  const double dt_e = args.dt;
  const R dt_r = (R)args.dt;

  // ---- constant Jacobian structure (written once) ----
  if constexpr (M::kLinearParams) {
    for (int e = lane; e < NX * NX; e += G) As[(e / NX) * LDA + e % NX] = thg[e];
    for (int e = lane; e < NX * NU; e += G) Bs[e] = thg[NX * NX + e];
  } else {
    M::template jac_const<R>(th_r, dt_r, As, LDA, Bs, lane, G);
  }

  // ---- load x0, U_warm (clipped, ilqr.py:165); zero K, k (Workspace init) ----
  double umin[NU], umax[NU];
#pragma unroll
  for (int r = 0; r < NU; r++) {
    umin[r] = args.u_min[r];
    umax[r] = args.u_max[r];
  }
  {
    const R* xg = (const R*)args.x0 + (size_t)pid * NX;
    for (int e = lane; e < NX; e += G) Xn[e] = (double)xg[e];
    const R* ug = (const R*)args.U_warm + (size_t)pid * T * NU;
    for (int e = lane; e < T * NU; e += G) {
      double v = (double)ug[e];
      const int r = e % NU;
      const double lo = args.u_min[r], hi = args.u_max[r];
      v = v < lo ? lo : v;  // np.clip
      v = v > hi ? hi : v;
      Un[e] = v;
      kg[e] = 0.0;
    }
    for (int e = lane; e < T * NU * NX; e += G) Kg[e] = R(0);
  }
  __syncwarp(gm);

  auto stage_C = [&](int t, int buf) {
    const R* src = Cg + (size_t)t * NCS;
    R* dst = Cb + buf * NCS;
    for (int e = lane; e < NCS; e += G) cp_async_elem(dst + e, src + e);
    const R* s2 = cg + (size_t)t * NZ;
    R* d2 = cb + buf * NZ;
    for (int e = lane; e < NZ; e += G) cp_async_elem(d2 + e, s2 + e);
    cp_async_commit();
  };

  // stage cost 0.5 z'Cz + c'z of a trajectory point in double; rows of the dense
  // quadratic form are split over the LCX lanes of a slot (j = lane in slot) and
  // reduced with xor shuffles (every lane ends with the identical sum).
  auto stage_cost = [&](auto lcx_tag, const R* Cs, const R* cs, const double* x, const double* u,
                        int j, unsigned smask) -> double {
    constexpr int LCX = decltype(lcx_tag)::value;
    double z[NZ];
#pragma unroll
    for (int i = 0; i < NX; i++) z[i] = x[i];
#pragma unroll
    for (int i = 0; i < NU; i++) z[NX + i] = u[i];
    double part = 0.0;
    if constexpr (DIAG) {
      // _stage_cost_xu with a diagonal C: row_i = d_i z_i (kernels.py:133-145)
#pragma unroll
      for (int i = 0; i < NZ; i++) part += 0.5 * z[i] * ((double)Cs[i] * z[i]) + (double)cs[i] * z[i];
      return part;
    } else {
      constexpr int NR = (NZ + LCX - 1) / LCX;
#pragma unroll
      for (int m = 0; m < NR; m++) {
        const int i = j + m * LCX;
        if (i < NZ) {
          double row = 0.0;
          const R* Ci = Cs + i * NZ;
#pragma unroll
          for (int jj = 0; jj < NZ; jj++) row += (double)Ci[jj] * z[jj];
          double zi = 0.0;
#pragma unroll
          for (int k = 0; k < LCX; k++)
            if (j == k && k + m * LCX < NZ) zi = z[k + m * LCX];
          part += 0.5 * zi * row + (double)cs[i] * zi;
        }
      }
#pragma unroll
      for (int off = LCX / 2; off > 0; off >>= 1) part += __shfl_xor_sync(smask, part, off, G);
      return part;
    }
  };

  double J = 0.0;
  int active = 1, fail_t = -1, iterations = 0, converged = 0, diverged = 0;
  R* ahist = args.alpha_hist ? (R*)args.alpha_hist + (size_t)pid * args.K_max : nullptr;
  R* jhist = args.J_hist ? (R*)args.J_hist + (size_t)pid * (args.K_max + 1) : nullptr;
  if (ahist)
    for (int e = lane; e < args.K_max; e += G) ahist[e] = R(0);

  // =========================== initial rollout (kernels.py:161-178) ===========
  {
    double xc[NX];
#pragma unroll
    for (int i = 0; i < NX; i++) xc[i] = Xn[i];
    stage_C(0, 0);
    for (int t = 0; t < T; t++) {
      const int buf = t & 1;
      if (t + 1 < T) {
        stage_C(t + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        cp_async_wait_all();
      }
      __syncwarp(gm);
      double u[NU];
#pragma unroll
      for (int r = 0; r < NU; r++) u[r] = Un[t * NU + r];
      J += stage_cost(std::integral_constant<int, G>{}, Cb + buf * NCS, cb + buf * NZ, xc, u, lane, gm);
      double xn[NX];
      step_e<M, R>(th_e, dt_e, As, Bs, xc, u, xn);
      bool fin = true;
#pragma unroll
      for (int i = 0; i < NX; i++) {
        fin &= finite_(xn[i]);
        xc[i] = xn[i];
      }
#pragma unroll
      for (int i = 0; i < NX; i++)
        if ((i % G) == lane) Xn[(t + 1) * NX + i] = xn[i];
      __syncwarp(gm);
      if (!fin) {
        fail_t = t;
        active = 0;
        J = INFINITY;
        diverged = 1;  // rollout_failed (ilqr.py:196-200)
        break;
      }
    }
    cp_async_wait_all();
    __syncwarp(gm);
  }
  if (jhist && lane == 0) jhist[0] = (R)J;

  // =============================== iterations ==================================
  int it = 0;
  for (; it < args.K_max && active; it++) {
    // ------------------- stage 1+2: fused linearise + Riccati sweep -------------
    R vxx[NX];  // row `lane` of V_xx (value Hessian), carried across stages
#pragma unroll
    for (int b = 0; b < NX; b++) vxx[b] = R(0);
    for (int e = lane; e < NX; e += G) Vxs[e] = R(0);
    stage_C(T - 1, (T - 1) & 1);
    for (int t = T - 1; t >= 0; t--) {
      const int buf = t & 1;
      if (t > 0) {
        stage_C(t - 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        cp_async_wait_all();
      }
      const R* Cs = Cb + buf * NCS;
      const R* cs = cb + buf * NZ;
      // nominal point and state-dependent Jacobian entries
      R xr[NX], ur[NU];
#pragma unroll
      for (int i = 0; i < NX; i++) xr[i] = (R)Xn[t * NX + i];
#pragma unroll
      for (int i = 0; i < NU; i++) ur[i] = (R)Un[t * NU + i];
      __syncwarp(gm);  // previous stage finished reading As/Bs/MA; staging visible
      if constexpr (!M::kLinearParams) M::template jac_vary<R>(th_r, dt_r, xr, ur, As, LDA, Bs);
#pragma unroll
      for (int i = 0; i < NZ; i++)
        if ((i % G) == lane) zs[i] = (i < NX) ? xr[i < NX ? i : 0] : ur[i >= NX ? i - NX : 0];
      __syncwarp(gm);
      // gz = C z + c ; qx = gz_x + A' Vx ; qu = gz_u + B' Vx   (kernels.py:395-410)
      R qx = R(0);
      if (lane < NX) {
        const int a = lane;
        R s = cs[a];
        if constexpr (DIAG) {
          s += Cs[a] * zs[a];
        } else {
#pragma unroll
          for (int b = 0; b < NZ; b++) s += Cs[a * NZ + b] * zs[b];
        }
#pragma unroll
        for (int b = 0; b < NX; b++) s += As[b * LDA + a] * Vxs[b];
        qx = s;
      }
      if (lane < NU) {
        const int a = lane;
        R s = cs[NX + a];
        if constexpr (DIAG) {
          s += Cs[NX + a] * zs[NX + a];
        } else {
#pragma unroll
          for (int b = 0; b < NZ; b++) s += Cs[(NX + a) * NZ + b] * zs[b];
        }
#pragma unroll
        for (int b = 0; b < NX; b++) s += Bs[b * NU + a] * Vxs[b];
        qus[a] = s;
      }
      // MA = Vxx A, NB = Vxx B (row `lane`)
      if (lane < NX) {
        R ma[NX], nb[NU];
#pragma unroll
        for (int b = 0; b < NX; b++) ma[b] = R(0);
#pragma unroll
        for (int b = 0; b < NU; b++) nb[b] = R(0);
#pragma unroll
        for (int r = 0; r < NX; r++) {
          const R v = vxx[r];
#pragma unroll
          for (int b = 0; b < NX; b++) ma[b] += v * As[r * LDA + b];
#pragma unroll
          for (int b = 0; b < NU; b++) nb[b] += v * Bs[r * NU + b];
        }
#pragma unroll
        for (int b = 0; b < NX; b++) MA[lane * LDA + b] = ma[b];
#pragma unroll
        for (int b = 0; b < NU; b++) NB[lane * NU + b] = nb[b];
      }
      __syncwarp(gm);
      // Quu = C_uu + B' NB (kernels.py:434-439)
      for (int e = lane; e < NU * NU; e += G) {
        const int i = e / NU, j = e % NU;
        R s;
        if constexpr (DIAG) {
          s = (i == j) ? Cs[NX + i] : R(0);
        } else {
          s = Cs[(NX + i) * NZ + NX + j];
        }
#pragma unroll
        for (int r = 0; r < NX; r++) s += Bs[r * NU + i] * NB[r * NU + j];
        Quus[e] = s;
      }
      // Qux column `lane` (kernels.py:428-433) and Qxx row `lane` (kernels.py:422-427)
      R quxc[NU], qxx[NX];
      if (lane < NX) {
        const int b = lane;
#pragma unroll
        for (int i = 0; i < NU; i++) {
          R s;
          if constexpr (DIAG) {
            s = R(0);
          } else {
            s = Cs[(NX + i) * NZ + b];
          }
#pragma unroll
          for (int r = 0; r < NX; r++) s += Bs[r * NU + i] * MA[r * LDA + b];
          quxc[i] = s;
        }
        const int a = lane;
#pragma unroll
        for (int bb = 0; bb < NX; bb++) {
          if constexpr (DIAG) {
            qxx[bb] = (bb == a) ? Cs[a] : R(0);
          } else {
            qxx[bb] = Cs[a * NZ + bb];
          }
        }
#pragma unroll
        for (int r = 0; r < NX; r++) {
          const R ar = As[r * LDA + a];
#pragma unroll
          for (int bb = 0; bb < NX; bb++) qxx[bb] += ar * MA[r * LDA + bb];
        }
      }
      __syncwarp(gm);
      // ---- stage QP on the control increment (double, all lanes redundantly) ----
      double Quu_d[NU][NU], qu_d[NU], lo[NU], hi[NU], du[NU];
      bool fr[NU];
      Chol<NU> ch;
#pragma unroll
      for (int i = 0; i < NU; i++) {
#pragma unroll
        for (int j = 0; j < NU; j++) Quu_d[i][j] = (double)Quus[i * NU + j];
        qu_d[i] = (double)qus[i];
        const double un = Un[t * NU + i];
        lo[i] = umin[i] - un;
        hi[i] = umax[i] - un;
      }
      const bool ok = stage_qp<NU>(Quu_d, qu_d, lo, hi, args.boxqp_max_iter, args.boxqp_tol, du, fr, ch);
      if (!ok) {
        fail_t = t;
        active = 0;
        break;
      }
      // k_t = du (all dims, kernels.py:478); K rows of free dims (kernels.py:481-489)
      if (lane < NU) {
#pragma unroll
        for (int i = 0; i < NU; i++)
          if (i == lane) kg[t * NU + i] = du[i];
      }
      R kcol[NU];
      if (lane < NX) {
        const int b = lane;
        double rhs[NU], sol[NU];
#pragma unroll
        for (int i = 0; i < NU; i++) rhs[i] = fr[i] ? (double)quxc[i] : 0.0;
        chol_solve<NU>(ch, rhs, sol);
#pragma unroll
        for (int i = 0; i < NU; i++) {
          kcol[i] = fr[i] ? (R)(-sol[i]) : R(0);
          Kg[(t * NU + i) * NX + b] = kcol[i];
          KT[b * NU + i] = kcol[i];
          QuxT[b * NU + i] = quxc[i];
        }
        // (Quu K)[:, b] with the unregularised Quu (kernels.py:503-506)
#pragma unroll
        for (int i = 0; i < NU; i++) {
          R s = R(0);
#pragma unroll
          for (int q = 0; q < NU; q++) s += Quus[i * NU + q] * kcol[q];
          QuuKT[b * NU + i] = s;
        }
        // Vx update (kernels.py:491-498)
        R kt[NU];
#pragma unroll
        for (int i = 0; i < NU; i++) kt[i] = (R)du[i];
        R s = qx;
#pragma unroll
        for (int r = 0; r < NU; r++) {
          R rowq = R(0);
#pragma unroll
          for (int q = 0; q < NU; q++) rowq += Quus[r * NU + q] * kt[q];
          s += kcol[r] * (rowq + qus[r]) + quxc[r] * kt[r];
        }
        Vxs[b] = s;  // all lanes finished reading Vx (qx/qu) before the last sync
      }
      __syncwarp(gm);
      // Vxx update row `lane` (kernels.py:499-507), then symmetrise (kernels.py:510-512)
      if (lane < NX) {
        const int a = lane;
#pragma unroll
        for (int bb = 0; bb < NX; bb++) {
          R s = qxx[bb];
#pragma unroll
          for (int r = 0; r < NU; r++) {
            const R Kra = kcol[r], Qra = quxc[r];
            s += (Kra * QuuKT[bb * NU + r] + Kra * QuxT[bb * NU + r]) + Qra * KT[bb * NU + r];
          }
          MA[a * LDA + bb] = s;  // MA is dead after Qxx/Qux: reuse as the N buffer
        }
      }
      __syncwarp(gm);
      if (lane < NX) {
        const int a = lane;
#pragma unroll
        for (int bb = 0; bb < NX; bb++) vxx[bb] = R(0.5) * (MA[a * LDA + bb] + MA[bb * LDA + a]);
      }
    }
    cp_async_wait_all();
    __syncwarp(gm);

    // --------------------------- stage 3: line search ---------------------------
    const int slot = lane / LC, j = lane % LC;
    const unsigned smask = (LC == 32) ? 0xffffffffu
                                      : (((1u << LC) - 1u) << ((threadIdx.x & 31u) & ~(unsigned)(LC - 1)));
    double Jc[8];
    bool dead[8];
#pragma unroll
    for (int a = 0; a < 8; a++) {
      Jc[a] = 0.0;
      dead[a] = false;
    }
    if (active) {
      const int NA = args.n_alpha;
      for (int round = 0; round * NSLOT < NA; round++) {
        const int a_me = min(round * NSLOT + slot, NA - 1);
        const double alpha = args.alphas[a_me];
        double xc[NX];
#pragma unroll
        for (int i = 0; i < NX; i++) xc[i] = Xn[i];
        double Jm = 0.0;
        bool dm = false;
        stage_C(0, 0);
        for (int t = 0; t < T; t++) {
          const int buf = t & 1;
          if (t + 1 < T) {
            stage_C(t + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
          } else {
            cp_async_wait_all();
          }
          __syncwarp(gm);
          // feedback law u = clip(U + alpha k + K (x - X)) (kernels.py:560-568)
          constexpr int NUL = (NU + LC - 1) / LC;
          double urr[NUL];
#pragma unroll
          for (int rr = 0; rr < NUL; rr++) {
            const int r = j + rr * LC;
            double v = 0.0;
            if (r < NU) {
              v = Un[t * NU + r] + alpha * kg[t * NU + r];
              const R* Kr = Kg + (t * NU + r) * NX;
#pragma unroll
              for (int b = 0; b < NX; b++) v += (double)Kr[b] * (xc[b] - Xn[t * NX + b]);
              const double lo = args.u_min[r], hi = args.u_max[r];
              if (v < lo) v = lo;
              else if (v > hi) v = hi;
            }
            urr[rr] = v;
          }
          double u[NU];
#pragma unroll
          for (int r = 0; r < NU; r++)
            u[r] = __shfl_sync(smask, urr[r / LC], (lane & ~(LC - 1)) + (r % LC), G);
          Jm += stage_cost(std::integral_constant<int, LC>{}, Cb + buf * NCS, cb + buf * NZ, xc, u, j, smask);
          double xn[NX];
          step_e<M, R>(th_e, dt_e, As, Bs, xc, u, xn);
          bool fin = finite_(Jm);
#pragma unroll
          for (int i = 0; i < NX; i++) {
            fin &= finite_(xn[i]);
            xc[i] = xn[i];
          }
          dm |= !fin;  // dead candidates keep stepping (harmlessly) to stay in lockstep
          __syncwarp(gm);
        }
        cp_async_wait_all();
        if (dm) Jm = INFINITY;
#pragma unroll
        for (int s = 0; s < NSLOT; s++) {
          const double Js = __shfl_sync(gm, Jm, s * LC, G);
          const bool ds = __shfl_sync(gm, (int)dm, s * LC, G) != 0;
#pragma unroll
          for (int a = 0; a < 8; a++)
            if (a == round * NSLOT + s && a < NA) {
              Jc[a] = Js;
              dead[a] = ds;
            }
        }
        __syncwarp(gm);
      }
    }

    // ------------------------- epilogue (ilqr.py:216-244) -----------------------
    const int act = active;
    if (act) iterations = it + 1;
    int best = 0;
    double best_J = Jc[0];
    bool alld = dead[0];
#pragma unroll
    for (int a = 1; a < 8; a++) {
      if (a < args.n_alpha) {
        if (Jc[a] < best_J) {
          best_J = Jc[a];
          best = a;
        }
        alld = alld && dead[a];
      }
    }
    const bool all_dead = act && alld;
    const bool accept = act && !all_dead && (best_J < J);
    if (ahist && lane == 0) ahist[it] = accept ? (R)args.alphas[best] : R(0);
    if (accept) {
      // re-roll the winning candidate (bit-identical to its line-search pass) and
      // adopt it as the nominal trajectory; writes to X_t are delayed until the
      // feedback at t has read the old nominal X_t.
      const double alpha = args.alphas[best];
      double xc[NX];
#pragma unroll
      for (int i = 0; i < NX; i++) xc[i] = Xn[i];
      for (int t = 0; t < T; t++) {
        double v = 0.0;
        if (lane < NU) {
          const int r = lane;
          v = Un[t * NU + r] + alpha * kg[t * NU + r];
          const R* Kr = Kg + (t * NU + r) * NX;
#pragma unroll
          for (int b = 0; b < NX; b++) v += (double)Kr[b] * (xc[b] - Xn[t * NX + b]);
          const double lo = args.u_min[r], hi = args.u_max[r];
          if (v < lo) v = lo;
          else if (v > hi) v = hi;
        }
        double u[NU];
#pragma unroll
        for (int r = 0; r < NU; r++) u[r] = __shfl_sync(gm, v, r, G);
        __syncwarp(gm);
#pragma unroll
        for (int i = 0; i < NX; i++)
          if ((i % G) == lane) Xn[t * NX + i] = xc[i];
        if (lane < NU) Un[t * NU + lane] = v;
        double xn[NX];
        step_e<M, R>(th_e, dt_e, As, Bs, xc, u, xn);
#pragma unroll
        for (int i = 0; i < NX; i++) xc[i] = xn[i];
      }
#pragma unroll
      for (int i = 0; i < NX; i++)
        if ((i % G) == lane) Xn[T * NX + i] = xc[i];
      __syncwarp(gm);
    }
    const double J_prev = J;
    if (accept) J = best_J;
    if (all_dead) {
      diverged = 1;
      active = 0;
    }
    const double rel = fabs(J_prev - J) / fmax(1.0, fabs(J_prev));
    const bool no_step = act && !all_dead && !accept;
    const bool conv_now = (act && !all_dead) && (no_step || rel <= args.conv_tol);
    if (conv_now) {
      converged = 1;
      active = 0;
    }
    if (jhist && lane == 0) jhist[it + 1] = (R)J;
  }
  if (jhist && lane == 0)
    for (int e = it + 1; e <= args.K_max; e++) jhist[e] = (R)J;

  // ================================ outputs ====================================
  const bool failed = fail_t >= 0 || diverged;
  {
    R* Xo = (R*)args.X + (size_t)pid * (T + 1) * NX;
    for (int e = lane; e < (T + 1) * NX; e += G) Xo[e] = (R)Xn[e];
    R* Uo = (R*)args.U + (size_t)pid * T * NU;
    for (int e = lane; e < T * NU; e += G) Uo[e] = (R)Un[e];
    if (args.clamped) {
      uint8_t* co = args.clamped + (size_t)pid * T * NU;
      for (int e = lane; e < T * NU; e += G) {
        const int r = e % NU;
        co[e] = (uint8_t)(Un[e] <= args.u_min[r] || Un[e] >= args.u_max[r]);
      }
    }
    if (args.K) {
      R* Ko = (R*)args.K + (size_t)pid * T * NU * NX;
      for (int e = lane; e < T * NU * NX; e += G) Ko[e] = Kg[e];
    }
    if (args.k) {
      R* ko = (R*)args.k + (size_t)pid * T * NU;
      for (int e = lane; e < T * NU; e += G) ko[e] = (R)kg[e];
    }
    if (lane == 0) {
      ((R*)args.J)[pid] = (R)J;
      if (args.iters) args.iters[pid] = iterations;
      if (args.converged) args.converged[pid] = (uint8_t)(converged && !failed);
      if (args.diverged) args.diverged[pid] = (uint8_t)diverged;
      if (args.fail_t) args.fail_t[pid] = fail_t;
    }
  }
}

}  // namespace dmpc

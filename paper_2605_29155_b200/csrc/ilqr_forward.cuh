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
// Shared-memory layout per problem (FwdLayout): nominal X/U and k (double), a shadow
// X/U (double) that the first line-search candidate writes its trajectory into (so
// accepting it is a pointer swap, no re-roll), the K_t staging buffer(s), the Riccati
// scratch (R) and the C_t staging buffer(s) (R). The gains K live in an L2-resident
// global workspace ([problem][t][n_u][LDA], written by the sweep, streamed back per
// stage by the line search), which keeps ~8.5 KB of shared memory per 13-state problem.
//
// Scheduling: a persistent grid (resident blocks only). Each G-lane group claims its next
// problem with one atomicAdd on a per-launch counter; a group whose problem converges early
// claims more work instead of idling until the slowest problem of its block is done.
#pragma once
#include <type_traits>

#include "riccati.cuh"

namespace dmpc {

#ifdef DMPC_NO_SYMSKIP
constexpr bool kSymSkip = false;
#else
constexpr bool kSymSkip = true;
#endif

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
  void* Kw;            // gain workspace (B, T, NU, LDA) of R
  void* Pw;            // packed cost records (B, T, REC) of R
  long long kw_stride, pw_stride;  // per-problem workspace strides (elements of R, 128-byte multiples)
  int* ctr;            // per-launch work counter (zeroed before the launch)
};

__host__ __device__ constexpr int align_up(int v, int a) { return (v + a - 1) / a * a; }

// per-group shared-memory stride: whole 128-byte lines + G banks (see launch.cuh plan())
template <class Lay>
__host__ __device__ constexpr int group_stride(int T, int G) {
  return (Lay::make(T).total + 127) / 128 * 128 + 4 * G;
}

// stage-record buffers of the forward's pipes: double-buffered in f32 (the dense record of
// the sweep / line search then arrives a whole stage ahead instead of half a stage; the
// 1.4 KB per problem does not change the register-bound occupancy), single in f64 dense
template <class M, bool DIAG, class R>
constexpr int fwd_nbuf() {
#ifdef DMPC_FWD_NB1
  return DIAG ? 2 : 1;
#else
  return (DIAG || sizeof(R) == 4) ? 2 : 1;
#endif
}

template <class M, bool DIAG, class R, bool LOCK = false>
struct FwdLayout {
  using D = Dims<M, DIAG, R>;
  static constexpr int NB = fwd_nbuf<M, DIAG, R>();
  // kXs: the alpha_0 line-search candidate writes its states to a second state buffer (the
  // shared memory the register-Jacobian models no longer spend on A_t / B_t) instead of over
  // the nominal, so a rejected alpha_0 needs no restoring re-roll. Measured (B=16384, T=10,
  // dense f32): fixed work 3.18 -> 2.82 ms, random costs 2.52 -> 2.46 ms, but the hover batch
  // 0.892 -> 0.900 ms (the extra 1.2 KB per problem); so only the warp-lockstep schedule
  // (fixed-work solves, long horizons) uses it.
  static constexpr bool kXs = LOCK && has_jac_regs<M>::value && !M::kLinearParams;
  int oPe, oPr, oXn, oXs, oUn, oUs, okg, oKb, total;
  RicLayout<M, DIAG, R> ric;
  __host__ __device__ static constexpr FwdLayout make(int T) {
    FwdLayout L{};
    int o = 0;
    L.oPe = o; o += align_up(M::NP * 8, 16);
    L.oPr = o; o += align_up(M::NP * (int)sizeof(R), 16);
    L.oXn = o; o += (T + 1) * D::XLD * 8;
    L.oXs = o; o += kXs ? (T + 1) * D::XLD * 8 : 0;
    L.oUn = o; o += T * D::ULD * 8;
    L.oUs = o; o += T * D::ULD * 8;
    L.okg = o; o += T * D::ULD * 8;
    o = align_up(o, 16);
    L.oKb = o; o += NB * D::NU * D::LDM * (int)sizeof(R);
    o = align_up(o, 16);
    // models with register-resident Jacobian rows never read a shared A_t / B_t copy here
    L.ric = RicLayout<M, DIAG, R>::make(o, !(has_jac_regs<M>::value && !M::kLinearParams));
    // the record buffers are the last array of the Riccati scratch: extra ones follow it
    L.total = align_up(L.ric.end + (NB - D::NBUF) * D::REC * (int)sizeof(R), 16);
    return L;
  }
};

// x+ = f(x,u) in double; the linear model reads its [A|B] copy from shared memory.
template <class M, class R>
DMPC_DEV void step_e(const double* P, double dt, const R* As, int lda, const R* Bs, int ldb,
                     const double* x, const double* u, double* o) {
  if constexpr (M::kLinearParams) {
#pragma unroll
    for (int i = 0; i < M::NX; i++) {
      R arow[M::NX], brow[M::NU];
      lds_row<M::NX>(As + i * lda, arow);
      lds_row<M::NU>(Bs + i * ldb, brow);
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M::NX; j++) acc += (double)arow[j] * x[j];
#pragma unroll
      for (int j = 0; j < M::NU; j++) acc += (double)brow[j] * u[j];
      o[i] = acc;
    }
  } else {
    M::template step<double>(P, dt, x, u, o);
  }
}

// dst[i] = v[i] for the entries i = j (mod S) this lane owns (lane j of S): a select chain per
// owned entry and one store, instead of N predicated stores
template <int N, int S>
DMPC_DEV void store_owned(double* dst, const double (&v)[N], int j) {
#pragma unroll
  for (int i0 = 0; i0 < N; i0 += S) {
    double val = v[i0];
#pragma unroll
    for (int l = 1; l < S; l++)
      if (i0 + l < N) val = (j == l) ? v[i0 + l] : val;
    if (i0 + j < N) dst[i0 + j] = val;
  }
}

// Feedback law v + K_r (x - xbar) in double (kernels.py:560-568) as two independent DFMA
// chains; the line search and the winner's re-roll share it, so the re-roll reproduces
// the candidate bit for bit.
template <int NX, class R>
DMPC_DEV double feedback(double v, const R (&krow)[NX], const double (&x)[NX], const double (&xbar)[NX]) {
  double v1 = 0.0;
#pragma unroll
  for (int b = 0; b < NX; b++) {
    if (b & 1) v1 += (double)krow[b] * (x[b] - xbar[b]);
    else v += (double)krow[b] * (x[b] - xbar[b]);
  }
  return v + v1;
}

// TC > 0: the horizon is the compile-time constant TC (args.T == TC), so every shared-memory
// offset and trip count below is a constant (the bench horizon T=10 is instantiated).
#ifdef DMPC_FWD_PROF
// -DDMPC_FWD_PROF (development aid): per-phase clock64 totals of every group, summed into
// g_fwd_prof (0 setup/claim, 1 initial rollout, 2 sweep, 3 line search, 4 epilogue, 5 outputs)
__device__ unsigned long long g_fwd_prof[8];
__device__ unsigned g_fwd_done;
#define FWD_MARK(k)                                                    \
  do {                                                                 \
    const long long n_ = clock64();                                    \
    if (lane == 0) atomicAdd(&g_fwd_prof[k], (unsigned long long)(n_ - tp_)); \
    tp_ = n_;                                                          \
  } while (0)
#else
#define FWD_MARK(k)
#endif

template <class M, int G, bool DIAG, class R, bool LOCK, int TC = 0>
#ifndef DMPC_FWD_MINB
#define DMPC_FWD_MINB 3
#endif
#ifndef DMPC_FWD_MAXT
#define DMPC_FWD_MAXT 128
#endif
__global__ void __launch_bounds__(DMPC_FWD_MAXT, sizeof(R) == 4 ? (G == 4 && M::NX > 8 ? 2 : (M::NX <= 8 ? 4 : DMPC_FWD_MINB)) : 2) ilqr_forward_kernel(const FwdArgs args) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  constexpr int LDA = D::LDA, LDB = D::LDB, ZLD = D::ZLD, XLD = D::XLD, ULD = D::ULD;
  constexpr int RPL = (NX + G - 1) / G;  // state rows owned by each lane
  constexpr int NSLOT = G >= 4 ? 4 : G;  // concurrent line-search candidates
  constexpr int LC = G / NSLOT;          // lanes per candidate slot
  using Lay = FwdLayout<M, DIAG, R, LOCK>;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int grp = threadIdx.x / G;
  const int lane = threadIdx.x % G;
  if (grp >= args.gpb) return;
  const unsigned wm = __activemask();  // the warp's groups (kernel entry: converged)
  const unsigned gm = group_mask<G>();
  const int T = TC > 0 ? TC : args.T;
  const Lay L = Lay::make(T);
  const int sstride = TC > 0 ? group_stride<Lay>(TC, G) : args.smem_stride;
  unsigned char* base = smem_raw + (size_t)grp * sstride;
  constexpr bool kXs = Lay::kXs;
  double* Xn = (double*)(base + L.oXn);  // nominal states (kXs: swapped with Xs on accept)
  double* Xs = kXs ? (double*)(base + L.oXs) : Xn;
  double* const Ubuf0 = (double*)(base + L.oUn);
  double* const Ubuf1 = (double*)(base + L.oUs);
  double* kg = (double*)(base + L.okg);
  R* Kb = (R*)(base + L.oKb);
  Ric<M, DIAG, R> S;
  S.bind(base, L.ric);
  // Every group claims its own next problem with one atomicAdd by its lane 0 and a
  // group-masked broadcast. (A warp-wide claim — one full-mask shuffle reached by the two
  // groups of a warp at different times, while the other group executes group-masked
  // collectives — intermittently lost the second group's problem; tools/stress.py small.)
  auto claim = [&]() -> int {
    int u = 0;
    if (lane == 0) u = atomicAdd(args.ctr, 1);
    return __shfl_sync(gm, u, 0, G);
  };

  // Lockstep (LOCK): the groups of a warp claim together, the iteration loop's
  // trip count is the warp's (a group whose problem is done idles until the other
  // finishes), and they claim again together. Free-running, a group that finishes claims
  // at once; the groups then drift apart (one rolling out a new problem while the other is
  // mid-iteration) and the warp issues each group's instructions separately. Measured
  // (B=16384, T=10, 13/4 dense f32): free is 3% faster on the hover batch (iteration
  // counts 3-4, lockstep idles a group for E[max]-E[it] = 0.3 iterations per pair);
  // lockstep is 5% faster on random costs (2-10 iterations) and 21% faster at conv_tol=0
  // (free: 14.8 active threads per warp instruction).
  auto wany = [&](bool v) -> bool {
    if constexpr (LOCK) return __any_sync(wm, v);
    else return v;
  };
#ifdef DMPC_FWD_PROF
  long long tp_ = clock64();
#endif
  for (int pid_ = claim(); wany(pid_ < args.B); pid_ = claim()) {
  const bool live = !LOCK || pid_ < args.B;
  const int pid = live ? pid_ : 0;  // a group past the end reads problem 0, writes nothing
  {
  double* Un = Ubuf0;  // nominal controls (swapped with the alpha_0 candidate's on accept)
  double* Us = Ubuf1;
  const R* Cg = (const R*)args.C + (size_t)pid * T * D::NCS;
  const R* cg = (const R*)args.c + (size_t)pid * T * NZ;
  R* Kw = (R*)args.Kw + (size_t)pid * args.kw_stride;
  R* Ko = args.K ? (R*)args.K + (size_t)pid * T * NU * NX : nullptr;
  // the initial rollout stages C_t / c_t element-wise from the caller's arrays and writes
  // them out as packed, 16-byte aligned records (Pw); every later sweep and line search
  // stages those with 16-byte copies
  R* Pw = (R*)args.Pw + (size_t)pid * args.pw_stride;  // (written only when live)
  constexpr int FNB = Lay::NB;
  CostPipe<M, DIAG, R, G, FNB> fwdp{&S, Cg, cg, T, lane, +1};
  CostPipe<M, DIAG, R, G, FNB> bwdp{&S, Cg, cg, T, lane, -1, nullptr, nullptr, Pw};
  CostPipe<M, DIAG, R, G, FNB> lsp{&S, Cg, cg, T, lane, +1, Kw, Kb, Pw};

  // ---- parameters (prepared: raw + reciprocals), kept in shared memory ----
  const R* thg = (const R*)args.theta + (size_t)args.theta_stride * pid;
  double* P_e = (double*)(base + L.oPe);
  R* P_r = (R*)(base + L.oPr);
  if constexpr (!M::kLinearParams) {
    if (lane == 0) {
      double th_e[M::NTH > 0 ? M::NTH : 1], pe[M::NP];
      R th_r[M::NTH > 0 ? M::NTH : 1], pr[M::NP];
#pragma unroll
      for (int i = 0; i < M::NTH; i++) {
        th_r[i] = thg[i];
        th_e[i] = (double)th_r[i];
      }
      M::template prep<double>(th_e, pe);
      M::template prep<R>(th_r, pr);
#pragma unroll
      for (int i = 0; i < M::NP; i++) {
        P_e[i] = pe[i];
        P_r[i] = pr[i];
      }
    }
    __syncwarp(gm);
  }
  const double dt_e = args.dt;
  const R dt_r = (R)args.dt;

  // ---- constant Jacobian structure (written once) ----
  if constexpr (M::kLinearParams) {
    for (int e = lane; e < NX * NX; e += G) S.As[(e / NX) * D::LDM + e % NX] = thg[e];
    for (int e = lane; e < NX * NU; e += G) S.Bs[(e / NU) * LDB + e % NU] = thg[NX * NX + e];
  } else if constexpr (!has_jac_regs<M>::value) {
    M::template jac_const<R>(P_r, dt_r, S.As, D::LDM, S.Bs, LDB, lane, G);
  }

  // ---- load x0, U_warm (clipped, ilqr.py:165); zero K, k (Workspace init) ----
  {
    const R* xg = (const R*)args.x0 + (size_t)pid * NX;
    for (int e = lane; e < NX; e += G) Xn[e] = (double)xg[e];
    const R* ug = (const R*)args.U_warm + (size_t)pid * T * NU;
#pragma unroll 4
    for (int e = lane; e < T * NU; e += G) {
      double v = (double)ug[e];
      const int t = e / NU, r = e % NU;
      const double lo = args.u_min[r], hi = args.u_max[r];
      v = v < lo ? lo : v;  // np.clip
      v = v > hi ? hi : v;
      Un[t * ULD + r] = v;
      kg[t * ULD + r] = 0.0;
    }
  }
  __syncwarp(gm);

  // stage cost 0.5 z'Cz + c'z in double (_stage_cost_xu, kernels.py:133-145); rows of the
  // dense quadratic form are split over the LCX lanes of a slot (j = lane in slot). Each
  // lane returns its share; callers sum the shares over the horizon and reduce once
  // (sum_lanes, below) — no shuffle chain per stage. Diagonal costs are computed whole by
  // every lane.
  auto stage_cost = [&](auto lcx_tag, const R* Cs, const R* cs, const double* x, const double* u,
                        int j, unsigned smask) -> double {
    [[maybe_unused]] constexpr int LCX = decltype(lcx_tag)::value;
    double z[NZ];
#pragma unroll
    for (int i = 0; i < NX; i++) z[i] = x[i];
#pragma unroll
    for (int i = 0; i < NU; i++) z[NX + i] = u[i];
    double part = 0.0;
    if constexpr (DIAG) {
      R d[NZ], cc[NZ];
      lds_row<NZ>(Cs, d);
      lds_row<NZ>(cs, cc);
#pragma unroll
      for (int i = 0; i < NZ; i++) part += 0.5 * z[i] * ((double)d[i] * z[i]) + (double)cc[i] * z[i];
      return part;
    } else {
      // rows i = j + m*LCX for the NF row sets every lane of the slot owns ...
      constexpr int NF = NZ / LCX, RE = NZ - NF * LCX;
      double zown[NF > 0 ? NF : 1];
#pragma unroll
      for (int m = 0; m < NF; m++) {
        const int i = j + m * LCX;
        R crow[NZ];
        lds_row<NZ>(Cs + i * ZLD, crow);
        double ra[4] = {0.0, 0.0, 0.0, 0.0};  // 4 independent DFMA chains
#pragma unroll
        for (int jj = 0; jj < NZ; jj++) ra[jj & 3] += (double)crow[jj] * z[jj];
        const double row = (ra[0] + ra[1]) + (ra[2] + ra[3]);
        double zi = z[m * LCX];
#pragma unroll
        for (int k = 1; k < LCX; k++) zi = j == k ? z[k + m * LCX] : zi;
        zown[m] = zi;
        part += 0.5 * zi * row + (double)cs[i] * zi;
      }
      // ... and the RE < LCX leftover rows r split by COLUMNS over the slot's lanes (lane j
      // takes the columns of its own rows plus leftover column NF*LCX + j), instead of one
      // more full row pass in which only RE lanes of the slot work
#pragma unroll
      for (int e = 0; e < RE; e++) {
        constexpr int r0 = NF * LCX;
        const int r = r0 + e;
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < NF; m++) acc += (double)Cs[r * ZLD + j + m * LCX] * zown[m];
        if (j < RE) {
          double zl = z[r0];
#pragma unroll
          for (int k = 1; k < RE; k++) zl = j == k ? z[r0 + k] : zl;
          acc += (double)Cs[r * ZLD + r0 + j] * zl;
        }
        part += 0.5 * z[r] * acc;
        if (j == 0) part += (double)cs[r] * z[r];
      }
      return part;
    }
  };
  auto sum_lanes = [&](auto lcx_tag, double part, unsigned smask) -> double {
    constexpr int LCX = decltype(lcx_tag)::value;
    if constexpr (!DIAG) {
#pragma unroll
      for (int off = LCX / 2; off > 0; off >>= 1) part += __shfl_xor_sync(smask, part, off, G);
    }
    return part;
  };

  double J = 0.0;
  bool csym = DIAG;  // every C_t of this problem symmetric (dense: checked in the rollout)
  int active = 1, fail_t = -1, iterations = 0, converged = 0, diverged = 0;
  int k_lo = T;  // gains output rows [k_lo, T) were written by some sweep
  R* ahist = args.alpha_hist && live ? (R*)args.alpha_hist + (size_t)pid * args.K_max : nullptr;
  R* jhist = args.J_hist && live ? (R*)args.J_hist + (size_t)pid * (args.K_max + 1) : nullptr;
  if (!live) active = 0;
  if (ahist)
    for (int e = lane; e < args.K_max; e += G) ahist[e] = R(0);

  FWD_MARK(0);
  // =========================== initial rollout (kernels.py:161-178) ===========
  if (live) {
    double xc[NX];
    lds_row_d<NX>(Xn, xc);
    fwdp.start(0);
    bool asym = false;
    for (int t = 0; t < T; t++) {
      fwdp.acquire(t);
      __syncwarp(gm);
      fwdp.pack_out(Pw, t);
      if constexpr (!DIAG && kSymSkip) {  // symmetric C: the value update needs no symmetrisation pass
        // lane a compares row a with column a (rows a + G, ... too): one vector row load,
        // NZ scalar column loads
        const R* Ct = fwdp.C(t);
#pragma unroll
        for (int a0 = 0; a0 < NZ; a0 += G) {
          const int a = a0 + lane;
          if (a < NZ) {
            R row[NZ];
            lds_row<NZ>(Ct + a * ZLD, row);
#pragma unroll
            for (int jj = 0; jj < NZ; jj++) asym |= !(row[jj] == Ct[jj * ZLD + a]);
          }
        }
      }
      double u[NU];
      lds_row_d<NU>(Un + t * ULD, u);
      J += stage_cost(std::integral_constant<int, G>{}, fwdp.C(t), fwdp.c(t), xc, u, lane, gm);  // lane share
      __syncwarp(gm);
      fwdp.release(t);
      double xn[NX];
      step_e<M, R>(P_e, dt_e, S.As, D::LDM, S.Bs, LDB, xc, u, xn);
      bool fin = true;
#pragma unroll
      for (int i = 0; i < NX; i++) {
        fin &= finite_(xn[i]);
        xc[i] = xn[i];
      }
      store_owned<NX, G>(Xn + (t + 1) * XLD, xn, lane);
      __syncwarp(gm);
      if (!fin) {
        fail_t = t;
        active = 0;
        diverged = 1;  // rollout_failed (ilqr.py:196-200)
        // rows past the failure keep the reference Workspace's zero init (ilqr.py:84-133),
        // not states of the group's previous problem
        for (int e = lane; e < (T - 1 - t) * XLD; e += G) Xn[(t + 2) * XLD + e] = 0.0;
        __syncwarp(gm);
        break;
      }
    }
    J = sum_lanes(std::integral_constant<int, G>{}, J, gm);
    if constexpr (!DIAG) csym = !__any_sync(gm, asym);
    if (fail_t >= 0) J = INFINITY;
    cp_async_wait_all();
    __syncwarp(gm);
  }
  if (jhist && lane == 0) jhist[0] = (R)J;

  FWD_MARK(1);
  // =============================== iterations ==================================
  int it = 0, passes = 0;
  for (; it < args.K_max && wany(active); it++) {
    if constexpr (LOCK) {
      if (!active) continue;  // done: wait for the warp's other groups
      passes++;
    }
    // ------------------- stage 1+2: fused linearise + Riccati sweep -------------
    R vxx[RPL][NX];  // the lane's rows of V_xx (value Hessian), carried across stages
#pragma unroll
    for (int k = 0; k < RPL; k++)
#pragma unroll
      for (int bb = 0; bb < NX; bb++) vxx[k][bb] = R(0);
    for (int e = lane; e < NX; e += G) S.Vx[e] = R(0);
    bwdp.start(T - 1);
    for (int t = T - 1; t >= 0; t--) {
      bwdp.acquire(t);
      const R* Cs = bwdp.C(t);
      const R* cs = bwdp.c(t);
      // nominal point, state-dependent Jacobian entries
      double ud[NU];
      lds_row_d<NU>(Un + t * ULD, ud);
      // z_t in the Riccati type: entry i converted once, by lane i (mod G)
#pragma unroll
      for (int k0 = 0; k0 < NZ; k0 += G) {
        const int i = k0 + lane;
        if (i < NZ) S.zs[i] = (R)*(i < NX ? Xn + t * XLD + i : Un + t * ULD + (i - NX));
      }
      __syncwarp(gm);  // previous stage done with As/Bs/MA; z_t and the staging visible
      R zv[NZ], vx[NX];
      lds_row<NZ>(S.zs, zv);
      // stage Jacobian values once: register rows for the products, plus the shared copy
      // of the state-dependent entries for the column accesses (A'Vx, B'NB)
      using Rows = std::conditional_t<has_jac_regs<M>::value, RegRows<M, R>, SmemRows<M, DIAG, R>>;
      Rows rows = make_rows<M, DIAG, R>(S, P_r, dt_r, zv);
      constexpr bool kRegJ = has_jac_regs<M>::value;
      if constexpr (kRegJ) {
        // A'Vx / B'Vx below are formed from the register rows: no shared copy needed
      } else if constexpr (!M::kLinearParams) {
        R xr[NX], ur[NU];
#pragma unroll
        for (int i = 0; i < NX; i++) xr[i] = zv[i];
#pragma unroll
        for (int i = 0; i < NU; i++) ur[i] = zv[NX + i];
        M::template jac_vary<R>(P_r, dt_r, xr, ur, S.As, D::LDM, S.Bs, LDB);
      }
      if constexpr (!kRegJ) __syncwarp(gm);
      // gz = C z + c ; qx = gz_x + A' Vx ; qu = gz_u + B' Vx   (kernels.py:395-410)
      R qx[RPL];
      lds_row<NX>(S.Vx, vx);
      // Register rows: column c of A' Vx as the same two FMA chains (even / odd rows b2, in
      // order, structural zeros skipped: +0 terms) the shared-copy products below form, so
      // the values are bit-identical; each lane keeps the columns it owns (selects).
      R avx[RPL][2], bvx[2];
      if constexpr (kRegJ) {
#pragma unroll
        for (int k = 0; k < RPL; k++) avx[k][0] = avx[k][1] = R(0);
        bvx[0] = bvx[1] = R(0);
#pragma unroll
        for (int cc = 0; cc < NX; cc++) {
          R e[2] = {R(0), R(0)};
#pragma unroll
          for (int b2 = 0; b2 < NX; b2++) {
            if (!M::a_nz(b2, cc)) continue;
            R arow[NX], brow[NU];
            rows.get(b2, arow, brow);
            if (M::a_one(b2, cc)) e[b2 & 1] += vx[b2];
            else if (M::a_dt(b2, cc)) e[b2 & 1] += dt_r * vx[b2];
            else e[b2 & 1] += arow[cc] * vx[b2];
          }
#pragma unroll
          for (int k = 0; k < RPL; k++) {
            const int a = min(row_of<G, RPL>(lane, k), NX - 1);
            avx[k][0] = a == cc ? e[0] : avx[k][0];
            avx[k][1] = a == cc ? e[1] : avx[k][1];
          }
        }
#pragma unroll
        for (int cc = 0; cc < NU; cc++) {
          R e[2] = {R(0), R(0)};
#pragma unroll
          for (int b2 = 0; b2 < NX; b2++)
            if (b_row_nz<M>(b2)) e[b2 & 1] += rows.b(b2, cc) * vx[b2];
          bvx[0] = lane == cc ? e[0] : bvx[0];
          bvx[1] = lane == cc ? e[1] : bvx[1];
        }
      }
#pragma unroll
      for (int k = 0; k < RPL; k++) {
        const int a = min(row_of<G, RPL>(lane, k), NX - 1);
        R sa[4] = {cs[a], R(0), R(0), R(0)};  // independent FMA chains
        if constexpr (DIAG) {
          sa[1] = Cs[a] * S.zs[a];
        } else {
          R crow[NZ];
          lds_row<NZ>(Cs + a * ZLD, crow);
#pragma unroll
          for (int b2 = 0; b2 < NZ; b2++) sa[b2 & 1] += crow[b2] * zv[b2];
        }
        if constexpr (kRegJ) {
          sa[2] = avx[k][0];
          sa[3] = avx[k][1];
        } else {
#pragma unroll
          for (int b2 = 0; b2 < NX; b2++) sa[2 + (b2 & 1)] += S.As[b2 * D::LDM + a] * vx[b2];
        }
        qx[k] = (sa[0] + sa[1]) + (sa[2] + sa[3]);
      }
      for (int a = lane; a < NU; a += G) {
        R sa[4] = {cs[NX + a], R(0), R(0), R(0)};
        if constexpr (DIAG) {
          sa[1] = Cs[NX + a] * S.zs[NX + a];
        } else {
          R crow[NZ];
          lds_row<NZ>(Cs + (NX + a) * ZLD, crow);
#pragma unroll
          for (int b2 = 0; b2 < NZ; b2++) sa[b2 & 1] += crow[b2] * zv[b2];
        }
        if constexpr (kRegJ) {
          sa[2] = bvx[0];
          sa[3] = bvx[1];
        } else {
#pragma unroll
          for (int b2 = 0; b2 < NX; b2++)
            if (b_row_nz<M>(b2)) sa[2 + (b2 & 1)] += S.Bs[b2 * LDB + a] * vx[b2];
        }
        S.qu[a] = (sa[0] + sa[1]) + (sa[2] + sa[3]);
      }
      ric_MA_NB<M, DIAG, R, G, RPL>(S, lane, vxx, dt_r, rows);
      __syncwarp(gm);
      for (int e = lane; e < NU * NU; e += G) S.Quu[(e / NU) * LDB + e % NU] = ric_Quu_entry<M, DIAG, R>(S, Cs, e / NU, e % NU, rows);
      R quxc[RPL][NU], qxx[RPL][NX];
      ric_Qxx_Qux<M, DIAG, R, G, RPL>(S, Cs, lane, qxx, quxc, dt_r, rows);
      __syncwarp(gm);
      bwdp.release(t);  // C_t fully consumed: prefetch C_{t-1}
      // ---- stage QP on the control increment (type R, all lanes redundantly) ----
      R quu[NU][NU], qu_c[NU], lo[NU], hi[NU], du[NU];
      bool fr[NU], lam0;
      Chol<NU, R> ch;
#pragma unroll
      for (int i = 0; i < NU; i++) {
        lds_row<NU>(S.Quu + i * LDB, quu[i]);
        qu_c[i] = S.qu[i];
        lo[i] = (R)(args.u_min[i] - ud[i]);
        hi[i] = (R)(args.u_max[i] - ud[i]);
      }
      const bool ok = stage_qp<NU, R>(quu, qu_c, lo, hi, args.boxqp_max_iter, (R)args.boxqp_tol, du, fr, ch, lam0);
      if (!ok) {
        fail_t = t;
        active = 0;
        break;
      }
      // k_t = du (all dims, kernels.py:478); K rows of free dims (kernels.py:481-489).
      // A coordinate the QP left on a bound is stored as the double-precision bound
      // offset (u_min - U_t or u_max - U_t), exactly the value the reference's boxQP
      // clamps to, so U_t + k_t lands on the bound bit-exactly (clamp masks match).
      {  // lane i < NU writes component i (selects instead of a lane-0 loop with branches)
        static_assert(NU <= G, "one lane per control component");
        const int i = lane < NU ? lane : 0;
        R dui = du[0], loi = lo[0], hii = hi[0];
        double udi = ud[0];
#pragma unroll
        for (int q = 1; q < NU; q++) {
          dui = i == q ? du[q] : dui;
          loi = i == q ? lo[q] : loi;
          hii = i == q ? hi[q] : hii;
          udi = i == q ? ud[q] : udi;
        }
        const double kd = dui <= loi ? args.u_min[i] - udi : (dui >= hii ? args.u_max[i] - udi : (double)dui);
        if (lane < NU) kg[t * ULD + lane] = kd;
      }
      R kcol[RPL][NU];
#pragma unroll
      for (int k = 0; k < RPL; k++) {
        const int b2 = row_of<G, RPL>(lane, k);
        R rhs[NU], sol[NU];
#pragma unroll
        for (int i = 0; i < NU; i++) rhs[i] = fr[i] ? quxc[k][i] : R(0);
        chol_solve<NU, R>(ch, rhs, sol);
#pragma unroll
        for (int i = 0; i < NU; i++) kcol[k][i] = fr[i] ? -sol[i] : R(0);
        if (b2 < NX) {
#pragma unroll
          for (int i = 0; i < NU; i++) Kw[(t * NU + i) * LDA + b2] = kcol[k][i];
          if (Ko) {  // the gains output holds the last computed K (ilqr.py:264)
#pragma unroll
            for (int i = 0; i < NU; i++) Ko[(t * NU + i) * NX + b2] = kcol[k][i];
          }
          ric_publish_cols<M, DIAG, R>(S, b2, kcol[k], quxc[k], lam0);
          // Vx update (kernels.py:491-498), unregularised Quu
          R s = qx[k];
#pragma unroll
          for (int r = 0; r < NU; r++) {
            R rowq = R(0);
#pragma unroll
            for (int q = 0; q < NU; q++) rowq += quu[r][q] * du[q];
            s += kcol[k][r] * (rowq + qu_c[r]) + quxc[k][r] * du[r];
          }
          S.Vx[b2] = s;  // all lanes finished reading Vx (qx/qu) before the last sync
        }
      }
      k_lo = t;
      __syncwarp(gm);
      if (kSymSkip && csym && lam0) {
        ric_Vxx_lean_regs<M, DIAG, R, G, RPL>(S, lane, qxx, quxc, vxx);
      } else {
        ric_Vxx_rows<M, DIAG, R, G, RPL>(S, lane, qxx, kcol, quxc, quu, lam0);
        __syncwarp(gm);
        ric_symmetrize<M, DIAG, R, G, RPL>(S, lane, vxx);
      }
    }
    cp_async_wait_all();
    __syncwarp(gm);

    FWD_MARK(2);
    // --------------------------- stage 3: line search ---------------------------
    const int slot = lane / LC, j = lane % LC;
    const unsigned smask = (LC == 32) ? 0xffffffffu
                                      : (((1u << LC) - 1u) << ((threadIdx.x & 31u) & ~(unsigned)(LC - 1)));
    // candidates are folded in increasing alpha index as they complete: the first
    // minimum wins ties (argmin, ilqr.py:218-222)
    double best_J = 0.0;
    int best = 0;
    bool alld = false;
    const bool inplace = args.n_alpha <= NSLOT;  // one round: alpha_0 may overwrite X
    if (active) {
      const int NA = args.n_alpha;
      for (int round = 0; round * NSLOT < NA; round++) {
        const int a_me = min(round * NSLOT + slot, NA - 1);
        const double alpha = args.alphas[a_me];
        double xc[NX];
        lds_row_d<NX>(Xn, xc);
        double Jm = 0.0;
        bool dm = false;
        // alpha_0 keeps its trajectory: controls in Us, states written over the nominal
        // X_t once every slot has read it (restored by a re-roll if alpha_0 loses)
        const bool shadow = inplace && (slot == 0);
        lsp.start(0);
        for (int t = 0; t < T; t++) {
          lsp.acquire(t);
          __syncwarp(gm);
          // feedback law u = clip(U + alpha k + K (x - X)) (kernels.py:560-568)
          constexpr int NUL = (NU + LC - 1) / LC;
          double xbar[NX];
          lds_row_d<NX>(Xn + t * XLD, xbar);
          double urr[NUL];
#pragma unroll
          for (int rr = 0; rr < NUL; rr++) {
            const int r = j + rr * LC;
            double v = 0.0;
            if (r < NU) {
              v = Un[t * ULD + r] + alpha * kg[t * ULD + r];
              R krow[NX];
              lds_row<NX>(lsp.K(t) + r * D::LDM, krow);
              v = feedback<NX>(v, krow, xc, xbar);
              const double lo = args.u_min[r], hi = args.u_max[r];
              if (v < lo) v = lo;
              else if (v > hi) v = hi;
              if (shadow) Us[t * ULD + r] = v;
            }
            urr[rr] = v;
          }
          double u[NU];
#pragma unroll
          for (int r = 0; r < NU; r++)
            u[r] = (LC == 1) ? urr[r] : __shfl_sync(smask, urr[r / LC], (lane & ~(LC - 1)) + (r % LC), G);
          Jm += stage_cost(std::integral_constant<int, LC>{}, lsp.C(t), lsp.c(t), xc, u, j, smask);
          __syncwarp(gm);  // every slot has read the nominal X_t
          if (shadow) store_owned<NX, LC>(Xs + t * XLD, xc, j);
          lsp.release(t);
          double xn[NX];
          step_e<M, R>(P_e, dt_e, S.As, D::LDM, S.Bs, LDB, xc, u, xn);
#pragma unroll
          for (int i = 0; i < NX; i++) xc[i] = xn[i];
          __syncwarp(gm);  // dead candidates keep stepping (harmlessly) to stay in lockstep
        }
        // dead candidates (kernels.py:569-574): a non-finite x_{t+1}, t < T-1, makes the
        // stage-(t+1) cost non-finite (z_i (C z)_i with z_i inf / nan; checked on the sum
        // below), and x_T, which no stage cost sees, is checked here: the reference's
        // per-stage tests, decided once per candidate
#pragma unroll
        for (int i = 0; i < NX; i++) dm |= !finite_(xc[i]);
        if (shadow) store_owned<NX, LC>(Xs + T * XLD, xc, j);
        cp_async_wait_all();
        // one reduction per candidate; a non-finite stage cost leaves a non-finite sum
        Jm = sum_lanes(std::integral_constant<int, LC>{}, Jm, smask);
        dm |= !finite_(Jm);
        if (dm) Jm = INFINITY;
#pragma unroll
        for (int s = 0; s < NSLOT; s++) {
          const double Js = __shfl_sync(gm, Jm, s * LC, G);
          const bool ds = __shfl_sync(gm, (int)dm, s * LC, G) != 0;
          const int a = round * NSLOT + s;
          if (a < NA) {
            if (a == 0) {
              best_J = Js;
              best = 0;
              alld = ds;
            } else {
              if (Js < best_J) {
                best_J = Js;
                best = a;
              }
              alld = alld && ds;
            }
          }
        }
        __syncwarp(gm);
      }
    }

    FWD_MARK(3);
    // ------------------------- epilogue (ilqr.py:216-244) -----------------------
    const int act = active;
    if (act) iterations = it + 1;
    const bool all_dead = act && alld;
    const bool accept = act && !all_dead && (best_J < J);
    if (ahist && lane == 0) ahist[it] = accept ? (R)args.alphas[best] : R(0);
    const bool inplace_used = act && inplace;  // alpha_0's states are in Xs (== X unless kXs)
    if (accept && best == 0 && inplace_used) {
      // adopt the alpha_0 candidate: its states are in Xs, its controls in Us
      __syncwarp(gm);
      double* tu = Un; Un = Us; Us = tu;
      if constexpr (kXs) {
        double* tx = Xn; Xn = Xs; Xs = tx;
      }
    } else if (accept || (!kXs && inplace_used)) {
      // Re-roll the nominal (xb, bit-identical to the rollout that produced it: restores X
      // after alpha_0 overwrote it; kXs: X is intact and xb is read from it) and, on accept, the winning candidate (xw, bit-identical
      // to its line-search pass), adopting the latter. Writes to X_t / U_t are delayed until
      // every lane has read the old U_t.
      const double alpha = args.alphas[best];
      double xw[NX], xb[NX];
      lds_row_d<NX>(Xn, xb);
#pragma unroll
      for (int i = 0; i < NX; i++) xw[i] = xb[i];
      constexpr int NUR = (NU + G - 1) / G;
      #pragma unroll 1
      for (int t = 0; t < T; t++) {
        double ub[NU];
        lds_row_d<NU>(Un + t * ULD, ub);
        double v[NUR], uw[NU];
#pragma unroll
        for (int r = 0; r < NU; r++) uw[r] = ub[r];
        if (accept) {
#pragma unroll
          for (int m2 = 0; m2 < NUR; m2++) {
            const int r = lane + m2 * G;
            v[m2] = 0.0;
            if (r < NU) {
              double w = Un[t * ULD + r] + alpha * kg[t * ULD + r];
              R krow[NX];
              if constexpr (sizeof(R) == 4) {
                const float4* kr4 = reinterpret_cast<const float4*>(Kw + (t * NU + r) * LDA);
#pragma unroll
                for (int q = 0; q < (NX + 3) / 4; q++) {
                  const float4 v4 = __ldcg(kr4 + q);
                  const float tt[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                  for (int i = 0; i < 4; i++)
                    if (q * 4 + i < NX) krow[q * 4 + i] = tt[i];
                }
              } else {
#pragma unroll
                for (int b = 0; b < NX; b++) krow[b] = __ldcg((const double*)(Kw + (t * NU + r) * LDA + b));
              }
              w = feedback<NX>(w, krow, xw, xb);
              const double lo = args.u_min[r], hi = args.u_max[r];
              if (w < lo) w = lo;
              else if (w > hi) w = hi;
              v[m2] = w;
            }
          }
#pragma unroll
          for (int r = 0; r < NU; r++) uw[r] = __shfl_sync(gm, v[r / G], r % G, G);
        }
        __syncwarp(gm);
#pragma unroll
        for (int i = 0; i < NX; i++)
          if ((i % G) == lane) Xn[t * XLD + i] = accept ? xw[i] : xb[i];
        if (accept) {
#pragma unroll
          for (int m2 = 0; m2 < NUR; m2++)
            if (lane + m2 * G < NU) Un[t * ULD + lane + m2 * G] = v[m2];
        }
        double xn[NX];
        if constexpr (kXs) {  // the nominal is intact (alpha_0 wrote to Xs): read, not re-rolled
          lds_row_d<NX>(Xn + (t + 1) * XLD, xb);
        } else {
          step_e<M, R>(P_e, dt_e, S.As, D::LDM, S.Bs, LDB, xb, ub, xn);
#pragma unroll
          for (int i = 0; i < NX; i++) xb[i] = xn[i];
        }
        if (accept) {
          step_e<M, R>(P_e, dt_e, S.As, D::LDM, S.Bs, LDB, xw, uw, xn);
#pragma unroll
          for (int i = 0; i < NX; i++) xw[i] = xn[i];
        }
      }
#pragma unroll
      for (int i = 0; i < NX; i++)
        if ((i % G) == lane) Xn[T * XLD + i] = accept ? xw[i] : xb[i];
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
    FWD_MARK(4);
  }
  if (jhist && lane == 0)
    for (int e = (LOCK ? passes : it) + 1; e <= args.K_max; e++) jhist[e] = (R)J;

  FWD_MARK(6);
  // ================================ outputs ====================================
  const bool failed = fail_t >= 0 || diverged;
  if (live) {
    R* Xo = (R*)args.X + (size_t)pid * (T + 1) * NX;
    #pragma unroll 1
    for (int e = lane; e < (T + 1) * NX; e += G) Xo[e] = (R)Xn[(e / NX) * XLD + e % NX];
    R* Uo = (R*)args.U + (size_t)pid * T * NU;
    #pragma unroll 1
    for (int e = lane; e < T * NU; e += G) Uo[e] = (R)Un[(e / NU) * ULD + e % NU];
    if (args.clamped) {
      uint8_t* co = args.clamped + (size_t)pid * T * NU;
      #pragma unroll 1
      for (int e = lane; e < T * NU; e += G) {
        const int r = e % NU;
        const double v = Un[(e / NU) * ULD + r];
        co[e] = (uint8_t)(v <= args.u_min[r] || v >= args.u_max[r]);
      }
    }
    if (Ko && k_lo > 0) {  // stages no sweep reached keep the zero-initialised gains
      #pragma unroll 1
      for (int e = lane; e < k_lo * NU * NX; e += G) Ko[e] = R(0);
    }
    if (args.k) {
      R* ko = (R*)args.k + (size_t)pid * T * NU;
      #pragma unroll 1
      for (int e = lane; e < T * NU; e += G) ko[e] = (R)kg[(e / NU) * ULD + e % NU];
    }
    if (lane == 0) {
      ((R*)args.J)[pid] = (R)J;
      if (args.iters) args.iters[pid] = iterations;
      if (args.converged) args.converged[pid] = (uint8_t)(converged && !failed);
      if (args.diverged) args.diverged[pid] = (uint8_t)diverged;
      if (args.fail_t) args.fail_t[pid] = fail_t;
    }
  }
  __syncwarp(gm);
  // (The workspace lines of a finished problem are NOT dropped with discard.global.L2: doing
  // so made ~100 of 16384 fixed-work solves differ run to run from their first iteration on,
  // while the write-back it saves is ~240 MB per launch, <2% of HBM time.)
  }  // problem scope
  FWD_MARK(5);
  }  // persistent loop
#ifdef DMPC_FWD_PROF
  if (lane == 0) {
    const unsigned done = atomicAdd(&g_fwd_done, 1u);
    if (done + 1 == gridDim.x * (unsigned)args.gpb) {
      printf("fwd prof (cycles, all groups): setup %llu rollout %llu sweep %llu linesearch %llu epilogue %llu "
             "outputs %llu after-loop %llu\n", g_fwd_prof[0], g_fwd_prof[1], g_fwd_prof[2], g_fwd_prof[3],
             g_fwd_prof[4], g_fwd_prof[5], g_fwd_prof[6]);
      for (int k = 0; k < 8; k++) g_fwd_prof[k] = 0;
      g_fwd_done = 0;
    }
  }
#endif
}

}  // namespace dmpc

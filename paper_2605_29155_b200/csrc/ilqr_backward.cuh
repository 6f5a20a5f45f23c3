// ilqr_backward.cuh — the fused implicit-differentiation backward kernel.
//
// One launch computes, per problem (group of G lanes, state on chip):
//   1. relinearisation at the solution and the clamp mask (U<=u_min)|(U>=u_max)
//      (MpcSolveLayer.backward, policy.py:257-272);
//   2. the auxiliary Riccati sweep whose linear cost is the seed, clamped control
//      dimensions frozen (kernels.py:582-707), giving dx0 = V_x after t = 0;
//   3. the differential rollout dX, dU (kernels.py:710-730) fused with the
//      gradient assembly dc = dz, dC = sym(dz z') (kernels.py:733-756), streamed
//      to HBM stage by stage with coalesced stores;
//   4. (NEW) the primal and auxiliary co-state recursions that give
//      the dynamics-parameter gradient, plus the optimal-cost (envelope) terms
//      scaled by dL/dJ.
// Everything runs in the ABI type R except the m x m Cholesky (double).
#pragma once
#include "ilqr_forward.cuh"

namespace dmpc {

struct BwdArgs {
  int B, T, theta_stride, n_theta, gpb, smem_stride;
  double dt;
  double u_min[8], u_max[8];
  const void* theta;
  const void* C;
  const void* c;
  const void* X;
  const void* U;
  const void* dLdX;
  const void* dLdU;
  const void* dLdJ;
  void* dC;
  void* dc;
  void* dx0;
  void* dtheta;
  void* dX;
  void* dU;
  int32_t* fail_t;
  void* Kg;  // lean layout: auxiliary gain workspace (B, T, NU, LDA) of R
  int ab;    // lean layout: the A_t / B_t region past each group's block is allocated
};

// Lean layout (models with register-resident Jacobian rows): the auxiliary gains K live in
// an L2 workspace (written by the sweep, streamed back one stage ahead by the rollout into
// two small staging buffers) and the shared A_t / B_t copy, which only the co-state
// recursions still use, sits past the end of the group's block and is allocated only when
// the call wants them (dtheta or dL/dJ): 9.2 -> 5.9 KB per 13-state problem, 4 blocks per SM.
template <class M>
constexpr bool bwd_lean() { return has_jac_regs<M>::value && !M::kLinearParams; }

template <class M, bool DIAG, class R>
struct BwdLayout {
  using D = Dims<M, DIAG, R>;
  static constexpr bool kLean = bwd_lean<M>();
  int oPr, oX, oU, oK, ok, odX, odU, ocl, olam, olh, oAB, total, total_ab;
  RicLayout<M, DIAG, R> ric;
  __host__ __device__ static constexpr BwdLayout make(int T) {
    BwdLayout L{};
    const int s = (int)sizeof(R);
    int o = 0;
    auto take = [&](int bytes) { int r = o; o = align_up(o + bytes, 16); return r; };
    L.oPr = take(M::NP * s);
    L.oX = take((T + 1) * D::LDA * s);
    L.oU = take(T * D::LDB * s);
    L.oK = take((kLean ? 2 : T) * D::NU * D::LDA * s);
    L.ok = take(T * D::LDB * s);
    L.odX = take((T + 1) * D::LDA * s);
    L.odU = take(T * D::LDB * s);
    L.ocl = take(T * D::NU);
    L.olam = take(D::LDA * s);
    L.olh = take(D::LDA * s);
    L.ric = RicLayout<M, DIAG, R>::make(o, !kLean);
    L.total = align_up(L.ric.end, 16);
    L.oAB = L.total;
    L.total_ab = kLean ? align_up(L.total + (D::NX * D::LDM + D::NX * D::LDB) * s, 16) : L.total;
    return L;
  }
};

// TC > 0: compile-time horizon (args.T == TC): constant shared-memory offsets (see the forward)
#ifndef DMPC_BWD_MINB
#define DMPC_BWD_MINB 3
#endif
template <class M, int G, bool DIAG, class R, int TC = 0>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? (G == 4 && M::NX > 8 ? 2 : (M::NX <= 8 || DIAG || bwd_lean<M>() ? 4 : DMPC_BWD_MINB)) : 2) ilqr_backward_kernel(const BwdArgs args) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  constexpr int LDA = D::LDA, LDB = D::LDB, ZLD = D::ZLD;
  constexpr int RPL = (NX + G - 1) / G;  // state rows owned by each lane
  using Lay = BwdLayout<M, DIAG, R>;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int grp = threadIdx.x / G;
  const int lane = threadIdx.x % G;
  const int pid = blockIdx.x * args.gpb + grp;
  if (grp >= args.gpb || pid >= args.B) return;
  const unsigned gm = group_mask<G>();
  const int T = TC > 0 ? TC : args.T;
  const Lay L = Lay::make(T);
  constexpr bool kLean = Lay::kLean;
  const int sstride = (TC > 0 && !kLean) ? group_stride<Lay>(TC, G) : args.smem_stride;
  unsigned char* base = smem_raw + (size_t)grp * sstride;
  R* Xs = (R*)(base + L.oX);    // rows of LDA
  R* Us = (R*)(base + L.oU);    // rows of LDB
  R* Ka = (R*)(base + L.oK);    // [t][r][LDA]
  R* ka = (R*)(base + L.ok);    // [t][LDB]
  R* dXs = (R*)(base + L.odX);  // rows of LDA
  R* dUs = (R*)(base + L.odU);  // rows of LDB
  uint8_t* cl = (uint8_t*)(base + L.ocl);
  R* lams = (R*)(base + L.olam);
  R* lhs = (R*)(base + L.olh);
  Ric<M, DIAG, R> S;
  S.bind(base, L.ric);
  if constexpr (kLean) {  // (only touched when args.ab: the co-state recursions)
    S.As = (R*)(base + L.oAB);
    S.Bs = S.As + D::NX * D::LDM;
  }
  R* const Kgp = kLean ? (R*)args.Kg + (size_t)pid * T * NU * LDA : nullptr;

  const R* Cg = (const R*)args.C + (size_t)pid * T * D::NCS;
  const R* cg = args.c ? (const R*)args.c + (size_t)pid * T * NZ : nullptr;
  const R* sXg = args.dLdX ? (const R*)args.dLdX + (size_t)pid * (T + 1) * NX : nullptr;
  const R* sUg = args.dLdU ? (const R*)args.dLdU + (size_t)pid * T * NU : nullptr;
  const R sJ = args.dLdJ ? ((const R*)args.dLdJ)[pid] : R(0);
  // the sweep's single pass over the caller's C: aligned block copies, unpadded rows (CLD)
  constexpr bool kBlk = !DIAG && D::NCS + 16 / (int)sizeof(R) - 1 <= D::NCSP;
  constexpr int CLD = kBlk ? NZ : ZLD;
  static_assert(DIAG || D::NCS + 16 / (int)sizeof(R) - 1 <= D::NBUF * D::REC, "dC staging holds the shifted block");
  CostPipe<M, DIAG, R, G, D::NBUF, kBlk> ricp{&S, Cg, nullptr, T, lane, -1};
  CostPipe<M, DIAG, R, G> adjp{&S, Cg, cg, T, lane, -1};
  const bool want_theta = args.dtheta != nullptr && args.n_theta > 0;
  const bool want_adjoint = want_theta || sJ != R(0);

  const R* thg = (const R*)args.theta + (size_t)args.theta_stride * pid;
  R* P_r = (R*)(base + L.oPr);
  if constexpr (!M::kLinearParams) {
    if (lane == 0) {
      R th_r[M::NTH > 0 ? M::NTH : 1], pr[M::NP];
#pragma unroll
      for (int i = 0; i < M::NTH; i++) th_r[i] = thg[i];
      M::template prep<R>(th_r, pr);
#pragma unroll
      for (int i = 0; i < M::NP; i++) P_r[i] = pr[i];
    }
    __syncwarp(gm);
  }
  const R dt_r = (R)args.dt;
  if constexpr (M::kLinearParams) {
    for (int e = lane; e < NX * NX; e += G) S.As[(e / NX) * D::LDM + e % NX] = thg[e];
    for (int e = lane; e < NX * NU; e += G) S.Bs[(e / NU) * LDB + e % NU] = thg[NX * NX + e];
  } else if (!kLean || args.ab) {
    M::template jac_const<R>(P_r, dt_r, S.As, D::LDM, S.Bs, LDB, lane, G);
  }
  {
    const R* xg = (const R*)args.X + (size_t)pid * (T + 1) * NX;
    // lane i takes column i of every row (rows unrolled for the compile-time horizon: all
    // the loads are in flight at once instead of one global latency per element)
#pragma unroll 11
    for (int t = 0; t <= T; t++) {
      for (int i = lane; i < NX; i += G) {
        Xs[t * LDA + i] = xg[t * NX + i];
        // the seeds dL/dX, dL/dU are parked in dX / dU (free until the differential
        // rollout) so the sweep reads them from shared memory, not global
        dXs[t * LDA + i] = sXg ? sXg[t * NX + i] : R(0);
      }
    }
    const R* ug = (const R*)args.U + (size_t)pid * T * NU;
#pragma unroll 4
    for (int e = lane; e < T * NU; e += G) {
      const R v = ug[e];
      const int t = e / NU, r = e % NU;
      Us[t * LDB + r] = v;
      dUs[t * LDB + r] = sUg ? sUg[e] : R(0);
      // clamped = (U <= u_min) | (U >= u_max)  (policy.py:271)
      cl[e] = (uint8_t)((double)v <= args.u_min[r] || (double)v >= args.u_max[r]);
    }
  }
  // V_x = dL/dX_T, V_xx = 0 (gradlayer.py:106-107)
  __syncwarp(gm);
  for (int e = lane; e < NX; e += G) S.Vx[e] = dXs[T * LDA + e];
  __syncwarp(gm);

  // ======================= auxiliary Riccati sweep (kernels.py:582-707) =========
  int fail_t = -1;
  {
    R vxx[RPL][NX];
#pragma unroll
    for (int k = 0; k < RPL; k++)
#pragma unroll
      for (int bb = 0; bb < NX; bb++) vxx[k][bb] = R(0);
    ricp.start(T - 1);
    for (int t = T - 1; t >= 0; t--) {
      ricp.acquire(t);
      const R* Cs = ricp.C(t);
      R xr[NX], ur[NU];
      lds_row<NX>(Xs + t * LDA, xr);
      lds_row<NU>(Us + t * LDB, ur);
      R zr[NZ];
#pragma unroll
      for (int i = 0; i < NX; i++) zr[i] = xr[i];
#pragma unroll
      for (int i = 0; i < NU; i++) zr[NX + i] = ur[i];
      __syncwarp(gm);
      // stage Jacobian values once (register rows + the shared copy for column accesses)
      using Rows = std::conditional_t<has_jac_regs<M>::value, RegRows<M, R>, SmemRows<M, DIAG, R>>;
      Rows rows = make_rows<M, DIAG, R>(S, P_r, dt_r, zr);
      constexpr bool kRegJ = has_jac_regs<M>::value;
      if constexpr (!kRegJ && !M::kLinearParams) {
        M::template jac_vary<R>(P_r, dt_r, xr, ur, S.As, D::LDM, S.Bs, LDB);
        __syncwarp(gm);
      }
      R qx[RPL];
      R vx[NX];
      lds_row<NX>(S.Vx, vx);
      if constexpr (kRegJ) {
        // A'Vx / B'Vx from the register rows (as in the forward sweep): every lane forms each
        // column's chain from its own seed, in the shared-copy products' order with the
        // structural zeros skipped (bit-identical), and keeps the column it owns
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int a = min(row_of<G, RPL>(lane, k), NX - 1);
          const R seed = dXs[t * LDA + a];
          R own = seed;
#pragma unroll
          for (int cc = 0; cc < NX; cc++) {
            R e = seed;
#pragma unroll
            for (int b2 = 0; b2 < NX; b2++) {
              if (!M::a_nz(b2, cc)) continue;
              R arow[NX], brow[NU];
              rows.get(b2, arow, brow);
              if (M::a_one(b2, cc)) e += vx[b2];
              else if (M::a_dt(b2, cc)) e += dt_r * vx[b2];
              else e += arow[cc] * vx[b2];
            }
            own = a == cc ? e : own;
          }
          qx[k] = own;
        }
        static_assert(!kRegJ || NU <= G, "one lane per control component");
        {
          const int a = lane < NU ? lane : 0;
          const R seed = dUs[t * LDB + a];
          R own = seed;
#pragma unroll
          for (int cc = 0; cc < NU; cc++) {
            R e = seed;
#pragma unroll
            for (int b2 = 0; b2 < NX; b2++)
              if (b_row_nz<M>(b2)) e += rows.b(b2, cc) * vx[b2];
            own = a == cc ? e : own;
          }
          if (lane < NU) S.qu[a] = own;
        }
      } else {
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int a = min(row_of<G, RPL>(lane, k), NX - 1);
          R s = dXs[t * LDA + a];
#pragma unroll
          for (int b2 = 0; b2 < NX; b2++) s += S.As[b2 * D::LDM + a] * vx[b2];
          qx[k] = s;
        }
        for (int a = lane; a < NU; a += G) {
          R s = dUs[t * LDB + a];
#pragma unroll
          for (int b2 = 0; b2 < NX; b2++) s += S.Bs[b2 * LDB + a] * vx[b2];
          S.qu[a] = s;
        }
      }
      ric_MA_NB<M, DIAG, R, G, RPL>(S, lane, vxx, dt_r, rows);
      __syncwarp(gm);
      for (int e = lane; e < NU * NU; e += G) S.Quu[(e / NU) * LDB + e % NU] = ric_Quu_entry<M, DIAG, R, CLD>(S, Cs, e / NU, e % NU, rows);
      R quxc[RPL][NU], qxx[RPL][NX];
      ric_Qxx_Qux<M, DIAG, R, G, RPL, CLD>(S, Cs, lane, qxx, quxc, dt_r, rows);
      __syncwarp(gm);
      ricp.release(t);
      // freeze clamped dimensions (kernels.py:658-667)
      R quu[NU][NU], qu[NU];
      bool clm[NU];
#pragma unroll
      for (int i = 0; i < NU; i++) {
        lds_row<NU>(S.Quu + i * LDB, quu[i]);
        qu[i] = S.qu[i];
        clm[i] = cl[t * NU + i] != 0;
      }
#pragma unroll
      for (int a = 0; a < NU; a++) {
        if (clm[a]) {
          qu[a] = R(0);
#pragma unroll
          for (int k = 0; k < RPL; k++) quxc[k][a] = R(0);
#pragma unroll
          for (int b2 = 0; b2 < NU; b2++) {
            quu[a][b2] = R(0);
            quu[b2][a] = R(0);
          }
          quu[a][a] = R(1);
        }
      }
      // full m x m Cholesky and the gains k = -Quu^-1 qu, K = -Quu^-1 Qux
      bool allf[NU];
#pragma unroll
      for (int i = 0; i < NU; i++) allf[i] = true;
      Chol<NU, R> ch;
      if (!chol_masked<NU, R>(quu, R(0), allf, ch)) {
        fail_t = t;
        break;
      }
      R kt[NU];
      {
        R sol[NU];
        chol_solve<NU, R>(ch, qu, sol);
#pragma unroll
        for (int i = 0; i < NU; i++) kt[i] = -sol[i];
      }
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < NU; i++) ka[t * LDB + i] = kt[i];
      }
      R kcol[RPL][NU];
#pragma unroll
      for (int k = 0; k < RPL; k++) {
        const int b2 = row_of<G, RPL>(lane, k);
        R sol[NU];
        chol_solve<NU, R>(ch, quxc[k], sol);
#pragma unroll
        for (int i = 0; i < NU; i++) kcol[k][i] = -sol[i];
        if (b2 < NX) {
#pragma unroll
          for (int i = 0; i < NU; i++) (kLean ? Kgp : Ka)[(t * NU + i) * LDA + b2] = kcol[k][i];
          ric_publish_cols<M, DIAG, R>(S, b2, kcol[k], quxc[k], true);
          R s = qx[k];
#pragma unroll
          for (int r = 0; r < NU; r++) {
            R rowq = R(0);
#pragma unroll
            for (int q = 0; q < NU; q++) rowq += quu[r][q] * kt[q];
            s += kcol[k][r] * (rowq + qu[r]) + quxc[k][r] * kt[r];
          }
          S.Vx[b2] = s;
        }
      }
      __syncwarp(gm);
      if constexpr (DIAG) {  // symmetric C: no symmetrisation pass needed (ric_Vxx_lean_regs)
        ric_Vxx_lean_regs<M, DIAG, R, G, RPL>(S, lane, qxx, quxc, vxx);
      } else {
        ric_Vxx_rows<M, DIAG, R, G, RPL>(S, lane, qxx, kcol, quxc, quu, true);
        __syncwarp(gm);
        ric_symmetrize<M, DIAG, R, G, RPL>(S, lane, vxx);
      }
    }
    cp_async_wait_all();
    __syncwarp(gm);
  }

  const bool failed = fail_t >= 0;
  R* dCo = args.dC ? (R*)args.dC + (size_t)pid * T * D::NCS : nullptr;
  R* dco = args.dc ? (R*)args.dc + (size_t)pid * T * NZ : nullptr;
  if (failed) {
    // failed instances get zero gradients (gradlayer.py:153-159, policy.py:277-280)
    if (dCo)
      for (int e = lane; e < T * D::NCS; e += G) dCo[e] = R(0);
    if (dco)
      for (int e = lane; e < T * NZ; e += G) dco[e] = R(0);
    if (args.dx0)
      for (int e = lane; e < NX; e += G) ((R*)args.dx0)[(size_t)pid * NX + e] = R(0);
    if (want_theta)
      for (int e = lane; e < args.n_theta; e += G) ((R*)args.dtheta)[(size_t)pid * args.n_theta + e] = R(0);
    __syncwarp(gm);
    for (int e = lane; e < (T + 1) * LDA; e += G) dXs[e] = R(0);  // (held the seeds)
    for (int e = lane; e < T * LDB; e += G) dUs[e] = R(0);
    __syncwarp(gm);
  } else {
    // ============ differential rollout + assembly (kernels.py:710-756) ============
    __syncwarp(gm);
    for (int e = lane; e < NX; e += G) dXs[e] = R(0);  // dX_0 = 0 (seeds no longer needed)
    __syncwarp(gm);
    // Models with register-resident Jacobian rows (JacRegs) propagate dx_{t+1} = A_t dx_t +
    // B_t du_t in registers: every lane forms the whole vector from compile-time rows (the
    // structural zeros skipped, the same FMA order as the row products over the shared copy,
    // so the values are bit-identical) -- no shared-memory A_t / B_t rewrite and reload per
    // stage, and dx stays in registers for the next stage.
    constexpr bool kRegJ = has_jac_regs<M>::value && !M::kLinearParams;
    R dxc[NX];
#pragma unroll
    for (int i = 0; i < NX; i++) dxc[i] = R(0);  // dX_0 = 0
    // lean layout: K_t arrives from the L2 workspace one stage ahead (16-byte copies into
    // the two staging buffers at Ka)
    constexpr int KCH = NU * LDA * (int)sizeof(R) / 16;
    auto issue_k = [&](int t) {
#pragma unroll
      for (int c0 = 0; c0 < KCH; c0 += G)
        if (c0 + lane < KCH)
          cp_async_16cg((char*)(Ka + (t & 1) * NU * LDA) + 16 * (c0 + lane), (const char*)(Kgp + (size_t)t * NU * LDA) + 16 * (c0 + lane));
      cp_async_commit();
    };
    if constexpr (kLean) {
      __threadfence_block();  // the sweep's gain stores before the group's copies of them
      __syncwarp(gm);
      issue_k(0);
    }
    for (int t = 0; t < T; t++) {
      if constexpr (kLean) {
        cp_async_wait_all();
        __syncwarp(gm);  // K_t resident; every lane done with the buffer K_{t+1} goes to
        if (t + 1 < T) issue_k(t + 1);
      }
      R xr[NX], ur[NU];
      lds_row<NX>(Xs + t * LDA, xr);
      lds_row<NU>(Us + t * LDB, ur);
      if constexpr (!M::kLinearParams && !kRegJ) M::template jac_vary<R>(P_r, dt_r, xr, ur, S.As, D::LDM, S.Bs, LDB);
      R dx[NX];
      if constexpr (kRegJ) {
#pragma unroll
        for (int i = 0; i < NX; i++) dx[i] = dxc[i];
      } else {
        lds_row<NX>(dXs + t * LDA, dx);
      }
      for (int r = lane; r < NU; r += G) {
        R s = ka[t * LDB + r];
        R krow[NX];
        lds_row<NX>(Ka + (kLean ? ((t & 1) * NU + r) : (t * NU + r)) * LDA, krow);
#pragma unroll
        for (int b = 0; b < NX; b++) s += krow[b] * dx[b];
        dUs[t * LDB + r] = s;
      }
      __syncwarp(gm);
      R du[NU];
      lds_row<NU>(dUs + t * LDB, du);
      if constexpr (kRegJ) {
        R z[NZ];
#pragma unroll
        for (int i = 0; i < NX; i++) z[i] = xr[i];
#pragma unroll
        for (int i = 0; i < NU; i++) z[NX + i] = ur[i];
        RegRows<M, R> rows;
        M::template jac_regs<R>(P_r, dt_r, z, rows.J);
#pragma unroll
        for (int a = 0; a < NX; a++) {
          R arow[NX], brow[NU];
          rows.get(a, arow, brow);
          R s = R(0);
#pragma unroll
          for (int b = 0; b < NX; b++) {
            if (M::a_one(a, b)) s += dx[b];
            else if (M::a_dt(a, b)) s += dt_r * dx[b];
            else if (M::a_nz(a, b)) s += arow[b] * dx[b];
          }
#pragma unroll
          for (int b = 0; b < NU; b++)
            if (M::b_nz(a, b)) s += brow[b] * du[b];
          dxc[a] = s;
        }
        // the lane's entries of dX_{t+1} (rows a = lane + k G) for the assembly and the output
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          R own = dxc[k * G];
#pragma unroll
          for (int l = 1; l < G; l++)
            if (k * G + l < NX) own = (lane == l) ? dxc[k * G + l] : own;
          if (k * G + lane < NX) dXs[(t + 1) * LDA + k * G + lane] = own;
        }
      }
#pragma unroll
      for (int k = 0; k < (kRegJ ? 0 : RPL); k++) {
        const int a = row_of<G, RPL>(lane, k);
        if (a < NX) {
          R arow[NX], brow[NU];
          lds_row<NX>(S.As + a * D::LDM, arow);
          lds_row<NU>(S.Bs + a * LDB, brow);
          R s = R(0);
#pragma unroll
          for (int b = 0; b < NX; b++) s += arow[b] * dx[b];
#pragma unroll
          for (int b = 0; b < NU; b++) s += brow[b] * du[b];
          dXs[(t + 1) * LDA + a] = s;
        }
      }
      // assembly of stage t: dc = dz, dC = 0.5 (dz z' + z dz'), clamped rows/cols zero;
      // plus the optimal-cost terms sJ z and sJ/2 z z'. Lane a owns row a (rows a + G for
      // a < NZ - G): z, dz and the clamp mask are in registers with compile-time column
      // indices, so each entry is a few FMAs and one store (no index arithmetic).
      {
        R zr[NZ], dzr[NZ];
        bool clr[NZ];
#pragma unroll
        for (int i = 0; i < NX; i++) {
          zr[i] = xr[i];
          dzr[i] = dx[i];
          clr[i] = false;
        }
#pragma unroll
        for (int i = 0; i < NU; i++) {
          zr[NX + i] = ur[i];
          dzr[NX + i] = du[i];
          clr[NX + i] = cl[t * NU + i] != 0;
        }
        // dense dC: lane a < G forms row a and mirrors its entries of the columns >= G into
        // rows >= G (dC is exactly symmetric: the same two rounded products, summed in either
        // order); only the (NZ-G)^2 corner is formed separately -- no second pass of all G
        // lanes for the NZ - G rows beyond the group width
        constexpr int NE = (!DIAG && NZ > G) ? NZ - G : 0;
        // the block is assembled in the (free) cost staging buffer at the alignment offset of
        // its global destination, so the copy-out below moves aligned 16-byte chunks
        R* blk = (!DIAG && dCo) ? dCo + (size_t)t * NZ * NZ : nullptr;
        R* Rd = S.Rb + (kBlk && blk ? blk_off(blk) : 0);
#pragma unroll
        for (int ce = 0; ce < NE * NE; ce++) {
          const int r = G + ce / (NE > 0 ? NE : 1), q = G + ce % (NE > 0 ? NE : 1);
          if (dCo && lane == ce % G) {
            const bool cq = clr[q], crr = clr[r];
            const R v = (crr || cq) ? R(0) : R(0.5) * (mul_rn(dzr[r], zr[q]) + mul_rn(zr[r], dzr[q]));
            Rd[r * NZ + q] = v + (R(0.5) * sJ * zr[r]) * zr[q];
          }
        }
#pragma unroll
        for (int e = 0; e < NE; e++)
          if (dco && lane == e) dco[t * NZ + G + e] = (clr[G + e] ? R(0) : dzr[G + e]) + sJ * zr[G + e];
#pragma unroll
        for (int k2 = 0; k2 < (NE > 0 ? 1 : (NZ + G - 1) / G); k2++) {
          const int a = lane + k2 * G;
          if (a < NZ) {
            const bool isx = a < NX;
            const R za = isx ? Xs[t * LDA + a] : Us[t * LDB + (isx ? 0 : a - NX)];
            const R da = isx ? dXs[t * LDA + a] : dUs[t * LDB + (isx ? 0 : a - NX)];
            const bool ca = !isx && cl[t * NU + (isx ? 0 : a - NX)] != 0;
            if (dco) dco[t * NZ + a] = (ca ? R(0) : da) + sJ * za;
            if (dCo) {
              if constexpr (DIAG) {
                const R v = ca ? R(0) : R(0.5) * (da * za + za * da);
                dCo[t * NZ + a] = v + R(0.5) * sJ * za * za;
              } else {
                // row a of dC_t goes to the (free) cost staging buffer first; the group then
                // writes the whole NZ x NZ block with consecutive lanes on consecutive words
                R* row = Rd + a * NZ;
                const R hs = R(0.5) * sJ * za;
#pragma unroll
                for (int b = 0; b < NZ; b++) {
                  // products rounded separately (no FMA contraction) so dC is exactly symmetric
                  const R v = (ca || clr[b]) ? R(0) : R(0.5) * (mul_rn(da, zr[b]) + mul_rn(za, dzr[b]));
                  row[b] = v + hs * zr[b];
                  if (b >= G) Rd[b * NZ + a] = v + (R(0.5) * sJ * zr[b]) * za;  // mirror into row b
                }
              }
            }
          }
        }
        if constexpr (!DIAG) {
          if (dCo) {
            __syncwarp(gm);
            constexpr int N = NZ * NZ, VN = 16 / (int)sizeof(R);
            if constexpr (!kBlk) {
#pragma unroll
              for (int e0 = 0; e0 < N; e0 += G)
                if (e0 + lane < N) blk[e0 + lane] = Rd[e0 + lane];
            } else {
            const int h = (VN - blk_off(blk)) & (VN - 1), nv = (N - h) / VN;
            using V = std::conditional_t<sizeof(R) == 4, float4, double2>;
#pragma unroll
            for (int m = 0; m < (N / VN + G - 1) / G; m++) {
              const int k = lane + m * G;
              if (k < nv) *reinterpret_cast<V*>(blk + h + VN * k) = *reinterpret_cast<const V*>(Rd + h + VN * k);
            }
            if (lane < h) blk[lane] = Rd[lane];
            const int e = h + VN * nv + lane;
            if (lane < VN && e < N) blk[e] = Rd[e];
            }
          }
        }
      }
      __syncwarp(gm);
    }

    // ============ co-state recursions: dtheta and the envelope terms (NEW) ========
    R gth[M::NTH > 0 && !M::kLinearParams ? M::NTH : 1];
#pragma unroll
    for (int i = 0; i < (M::NTH > 0 && !M::kLinearParams ? M::NTH : 1); i++) gth[i] = R(0);
    constexpr int NZL = M::kLinearParams ? NZ : 1;
    R grow[RPL][NZL];  // linear model: the lane's rows of [dA | dB]
#pragma unroll
    for (int k = 0; k < RPL; k++)
#pragma unroll
      for (int i = 0; i < NZL; i++) grow[k][i] = R(0);
    if (want_adjoint) {
      for (int e = lane; e < NX; e += G) {
        lams[e] = R(0);
        lhs[e] = sXg ? sXg[T * NX + e] : R(0);
      }
      adjp.start(T - 1);
      for (int t = T - 1; t >= 0; t--) {
        adjp.acquire(t);
        R xr[NX], ur[NU], dx[NX], du[NU], lm[NX], lh[NX];
        lds_row<NX>(Xs + t * LDA, xr);
        lds_row<NU>(Us + t * LDB, ur);
        lds_row<NX>(dXs + t * LDA, dx);
        lds_row<NU>(dUs + t * LDB, du);
        lds_row<NX>(lams, lm);
        lds_row<NX>(lhs, lh);
        __syncwarp(gm);
        if constexpr (!M::kLinearParams) M::template jac_vary<R>(P_r, dt_r, xr, ur, S.As, D::LDM, S.Bs, LDB);
        __syncwarp(gm);
        if (want_theta) {
          if constexpr (M::kLinearParams) {
#pragma unroll
            for (int k = 0; k < RPL; k++) {
              const int i = min(row_of<G, RPL>(lane, k), NX - 1);
              const R lhi = lhs[i], lmi = lams[i], lsi = sJ * lams[i];
#pragma unroll
              for (int j2 = 0; j2 < NX; j2++) grow[k][j2] += lhi * xr[j2] + lmi * dx[j2] + lsi * xr[j2];
#pragma unroll
              for (int j2 = 0; j2 < NU; j2++) grow[k][NX + j2] += lhi * ur[j2] + lmi * du[j2] + lsi * ur[j2];
            }
          } else if constexpr (M::NTH > 0) {
            R lhe[NX];
#pragma unroll
            for (int i = 0; i < NX; i++) lhe[i] = lh[i] + sJ * lm[i];
            M::template theta_grad<R>(P_r, dt_r, xr, ur, dx, du, lhe, lm, gth);
          }
        }
        const R* Cs = adjp.C(t);
        const R* cs = adjp.c(t);
        R nl[RPL], nh[RPL];
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int a = min(row_of<G, RPL>(lane, k), NX - 1);
          R s1 = cg ? cs[a] : R(0);
          R s2 = sXg ? sXg[t * NX + a] : R(0);
          if constexpr (DIAG) {
            s1 += Cs[a] * Xs[t * LDA + a];
            s2 += Cs[a] * dXs[t * LDA + a];
          } else {
            R crow[NZ];
            lds_row<NZ>(Cs + a * ZLD, crow);
#pragma unroll
            for (int b = 0; b < NZ; b++) {
              const R zb = b < NX ? xr[b < NX ? b : 0] : ur[b >= NX ? b - NX : 0];
              const R db = b < NX ? dx[b < NX ? b : 0] : du[b >= NX ? b - NX : 0];
              s1 += crow[b] * zb;
              s2 += crow[b] * db;
            }
          }
#pragma unroll
          for (int b = 0; b < NX; b++) {
            const R ab = S.As[b * D::LDM + a];
            s1 += ab * lm[b];
            s2 += ab * lh[b];
          }
          nl[k] = s1;
          nh[k] = s2;
        }
        __syncwarp(gm);
        adjp.release(t);
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int a = row_of<G, RPL>(lane, k);
          if (a < NX) {
            lams[a] = nl[k];
            lhs[a] = nh[k];
          }
        }
        __syncwarp(gm);
      }
      cp_async_wait_all();
      __syncwarp(gm);
    }
    if (args.dx0) {
      R* o = (R*)args.dx0 + (size_t)pid * NX;
      for (int e = lane; e < NX; e += G) o[e] = S.Vx[e] + (want_adjoint ? sJ * lams[e] : R(0));
    }
    if (want_theta) {
      R* o = (R*)args.dtheta + (size_t)pid * args.n_theta;
      if constexpr (M::kLinearParams) {
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int a = row_of<G, RPL>(lane, k);
          if (a < NX) {
#pragma unroll
            for (int j2 = 0; j2 < NX; j2++) o[a * NX + j2] = grow[k][j2];
#pragma unroll
            for (int j2 = 0; j2 < NU; j2++) o[NX * NX + a * NU + j2] = grow[k][NX + j2];
          }
        }
      } else if constexpr (M::NTH > 0) {
        if (lane == 0)
          for (int i = 0; i < M::NTH; i++) o[i] = gth[i];
      }
    }
  }
  if (args.dX)
    for (int e = lane; e < (T + 1) * NX; e += G)
      ((R*)args.dX)[(size_t)pid * (T + 1) * NX + e] = dXs[(e / NX) * LDA + e % NX];
  if (args.dU)
    for (int e = lane; e < T * NU; e += G)
      ((R*)args.dU)[(size_t)pid * T * NU + e] = dUs[(e / NU) * LDB + e % NU];
  if (args.fail_t && lane == 0) args.fail_t[pid] = fail_t;
}

}  // namespace dmpc

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
};

template <class M, bool DIAG, class R>
struct BwdLayout {
  static constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  static constexpr int LDA = NX;
  static constexpr int NCS = DIAG ? NZ : NZ * NZ;
  int oX, oU, oK, ok, odX, odU, ocl, oAs, oBs, oMA, oNB, oKT, oQuxT, oQuuKT, oqu, oVx, olam, olh,
      oC, oc, total;
  __host__ __device__ static BwdLayout make(int T) {
    BwdLayout L;
    const int s = (int)sizeof(R);
    int o = 0;
    L.oX = o; o += (T + 1) * NX * s;
    L.oU = o; o += T * NU * s;
    L.oK = o; o += T * NU * NX * s;
    L.ok = o; o += T * NU * s;
    L.odX = o; o += (T + 1) * NX * s;
    L.odU = o; o += T * NU * s;
    L.ocl = o; o += align_up(T * NU, 8);
    o = align_up(o, 16);
    L.oAs = o; o += NX * LDA * s;
    L.oBs = o; o += NX * NU * s;
    L.oMA = o; o += NX * LDA * s;
    L.oNB = o; o += NX * NU * s;
    L.oKT = o; o += NX * NU * s;
    L.oQuxT = o; o += NX * NU * s;
    L.oQuuKT = o; o += NX * NU * s;
    L.oqu = o; o += NU * s;
    L.oVx = o; o += NX * s;
    L.olam = o; o += NX * s;
    L.olh = o; o += NX * s;
    o = align_up(o, 16);
    L.oC = o; o += 2 * NCS * s;
    L.oc = o; o += 2 * NZ * s;
    L.total = align_up(o, 16);
    return L;
  }
};

template <class M, int G, bool DIAG, class R>
__global__ void __launch_bounds__(128) ilqr_backward_kernel(const BwdArgs args) {
  constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  using Lay = BwdLayout<M, DIAG, R>;
  constexpr int LDA = Lay::LDA, NCS = Lay::NCS;
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
  R* Xs = (R*)(base + L.oX);
  R* Us = (R*)(base + L.oU);
  R* Ka = (R*)(base + L.oK);
  R* ka = (R*)(base + L.ok);
  R* dXs = (R*)(base + L.odX);
  R* dUs = (R*)(base + L.odU);
  uint8_t* cl = (uint8_t*)(base + L.ocl);
  R* As = (R*)(base + L.oAs);
  R* Bs = (R*)(base + L.oBs);
  R* MA = (R*)(base + L.oMA);
  R* NB = (R*)(base + L.oNB);
  R* KT = (R*)(base + L.oKT);
  R* QuxT = (R*)(base + L.oQuxT);
  R* QuuKT = (R*)(base + L.oQuuKT);
  R* qus = (R*)(base + L.oqu);
  R* Vxs = (R*)(base + L.oVx);
  R* lams = (R*)(base + L.olam);
  R* lhs = (R*)(base + L.olh);
  R* Cb = (R*)(base + L.oC);
  R* cb = (R*)(base + L.oc);

  const R* Cg = (const R*)args.C + (size_t)pid * T * NCS;
  const R* cg = args.c ? (const R*)args.c + (size_t)pid * T * NZ : nullptr;
  const R* sXg = args.dLdX ? (const R*)args.dLdX + (size_t)pid * (T + 1) * NX : nullptr;
  const R* sUg = args.dLdU ? (const R*)args.dLdU + (size_t)pid * T * NU : nullptr;
  const R sJ = args.dLdJ ? ((const R*)args.dLdJ)[pid] : R(0);
  const bool want_theta = args.dtheta != nullptr && args.n_theta > 0;
  const bool want_adjoint = want_theta || sJ != R(0);

  const R* thg = (const R*)args.theta + (size_t)args.theta_stride * pid;
  R th_r[NTHL];
  if constexpr (!M::kLinearParams) {
#pragma unroll
    for (int i = 0; i < NTHL; i++) th_r[i] = (i < M::NTH) ? thg[i] : R(0);
  } else {
    th_r[0] = R(0);
  }
  const R dt_r = (R)args.dt;
  if constexpr (M::kLinearParams) {
    for (int e = lane; e < NX * NX; e += G) As[(e / NX) * LDA + e % NX] = thg[e];
    for (int e = lane; e < NX * NU; e += G) Bs[e] = thg[NX * NX + e];
  } else {
    M::template jac_const<R>(th_r, dt_r, As, LDA, Bs, lane, G);
  }
  {
    const R* xg = (const R*)args.X + (size_t)pid * (T + 1) * NX;
    for (int e = lane; e < (T + 1) * NX; e += G) {
      Xs[e] = xg[e];
      dXs[e] = R(0);
    }
    const R* ug = (const R*)args.U + (size_t)pid * T * NU;
    for (int e = lane; e < T * NU; e += G) {
      const R v = ug[e];
      const int r = e % NU;
      Us[e] = v;
      dUs[e] = R(0);
      // clamped = (U <= u_min) | (U >= u_max)  (policy.py:271)
      cl[e] = (uint8_t)((double)v <= args.u_min[r] || (double)v >= args.u_max[r]);
    }
  }
  auto stage_C = [&](int t, int buf) {
    const R* src = Cg + (size_t)t * NCS;
    R* dst = Cb + buf * NCS;
    for (int e = lane; e < NCS; e += G) cp_async_elem(dst + e, src + e);
    if (cg) {
      const R* s2 = cg + (size_t)t * NZ;
      R* d2 = cb + buf * NZ;
      for (int e = lane; e < NZ; e += G) cp_async_elem(d2 + e, s2 + e);
    }
    cp_async_commit();
  };
  auto load_z = [&](int t, R (&xr)[NX], R (&ur)[NU]) {
#pragma unroll
    for (int i = 0; i < NX; i++) xr[i] = Xs[t * NX + i];
#pragma unroll
    for (int i = 0; i < NU; i++) ur[i] = Us[t * NU + i];
  };
  // V_x = dL/dX_T, V_xx = 0 (gradlayer.py:106-107)
  for (int e = lane; e < NX; e += G) Vxs[e] = sXg ? sXg[T * NX + e] : R(0);
  __syncwarp(gm);

  // ======================= auxiliary Riccati sweep (kernels.py:582-707) =========
  int fail_t = -1;
  {
    R vxx[NX];
#pragma unroll
    for (int b = 0; b < NX; b++) vxx[b] = R(0);
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
      R xr[NX], ur[NU];
      load_z(t, xr, ur);
      __syncwarp(gm);
      if constexpr (!M::kLinearParams) M::template jac_vary<R>(th_r, dt_r, xr, ur, As, LDA, Bs);
      __syncwarp(gm);
      R qx = R(0);
      if (lane < NX) {
        const int a = lane;
        R s = sXg ? sXg[t * NX + a] : R(0);
#pragma unroll
        for (int b = 0; b < NX; b++) s += As[b * LDA + a] * Vxs[b];
        qx = s;
      }
      if (lane < NU) {
        const int a = lane;
        R s = sUg ? sUg[t * NU + a] : R(0);
#pragma unroll
        for (int b = 0; b < NX; b++) s += Bs[b * NU + a] * Vxs[b];
        qus[a] = s;
      }
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
      // Quu (all lanes, redundantly, into registers), Qux column, Qxx row
      R quu[NU][NU];
#pragma unroll
      for (int i = 0; i < NU; i++)
#pragma unroll
        for (int j = 0; j < NU; j++) {
          R s;
          if constexpr (DIAG) {
            s = (i == j) ? Cs[NX + i] : R(0);
          } else {
            s = Cs[(NX + i) * NZ + NX + j];
          }
#pragma unroll
          for (int r = 0; r < NX; r++) s += Bs[r * NU + i] * NB[r * NU + j];
          quu[i][j] = s;
        }
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
      // freeze clamped dimensions (kernels.py:658-667)
      R qu[NU];
#pragma unroll
      for (int i = 0; i < NU; i++) qu[i] = qus[i];
#pragma unroll
      for (int a = 0; a < NU; a++) {
        if (cl[t * NU + a]) {
          qu[a] = R(0);
          quxc[a] = R(0);
#pragma unroll
          for (int b = 0; b < NU; b++) {
            quu[a][b] = R(0);
            quu[b][a] = R(0);
          }
          quu[a][a] = R(1);
        }
      }
      __syncwarp(gm);
      // full m x m Cholesky (double) and the gains k = -Quu^-1 qu, K = -Quu^-1 Qux
      double Hd[NU][NU];
      bool allf[NU];
#pragma unroll
      for (int i = 0; i < NU; i++) {
        allf[i] = true;
#pragma unroll
        for (int j = 0; j < NU; j++) Hd[i][j] = (double)quu[i][j];
      }
      Chol<NU> ch;
      if (!chol_masked<NU>(Hd, allf, ch)) {
        fail_t = t;
        break;
      }
      R kt[NU];
      {
        double rhs[NU], sol[NU];
#pragma unroll
        for (int i = 0; i < NU; i++) rhs[i] = (double)qu[i];
        chol_solve<NU>(ch, rhs, sol);
#pragma unroll
        for (int i = 0; i < NU; i++) kt[i] = (R)(-sol[i]);
      }
      if (lane < NU) {
#pragma unroll
        for (int i = 0; i < NU; i++)
          if (i == lane) ka[t * NU + i] = kt[i];
      }
      R kcol[NU];
      if (lane < NX) {
        const int b = lane;
        double rhs[NU], sol[NU];
#pragma unroll
        for (int i = 0; i < NU; i++) rhs[i] = (double)quxc[i];
        chol_solve<NU>(ch, rhs, sol);
#pragma unroll
        for (int i = 0; i < NU; i++) {
          kcol[i] = (R)(-sol[i]);
          Ka[(t * NU + i) * NX + b] = kcol[i];
          KT[b * NU + i] = kcol[i];
          QuxT[b * NU + i] = quxc[i];
        }
#pragma unroll
        for (int i = 0; i < NU; i++) {
          R s = R(0);
#pragma unroll
          for (int q = 0; q < NU; q++) s += quu[i][q] * kcol[q];
          QuuKT[b * NU + i] = s;
        }
        R s = qx;
#pragma unroll
        for (int r = 0; r < NU; r++) {
          R rowq = R(0);
#pragma unroll
          for (int q = 0; q < NU; q++) rowq += quu[r][q] * kt[q];
          s += kcol[r] * (rowq + qu[r]) + quxc[r] * kt[r];
        }
        Vxs[b] = s;
      }
      __syncwarp(gm);
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
          MA[a * LDA + bb] = s;
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
  }

  const bool failed = fail_t >= 0;
  R* dCo = args.dC ? (R*)args.dC + (size_t)pid * T * (DIAG ? NZ : NZ * NZ) : nullptr;
  R* dco = args.dc ? (R*)args.dc + (size_t)pid * T * NZ : nullptr;
  if (failed) {
    // failed instances get zero gradients (gradlayer.py:153-159, policy.py:277-280)
    if (dCo)
      for (int e = lane; e < T * (DIAG ? NZ : NZ * NZ); e += G) dCo[e] = R(0);
    if (dco)
      for (int e = lane; e < T * NZ; e += G) dco[e] = R(0);
    if (args.dx0)
      for (int e = lane; e < NX; e += G) ((R*)args.dx0)[(size_t)pid * NX + e] = R(0);
    if (want_theta)
      for (int e = lane; e < args.n_theta; e += G) ((R*)args.dtheta)[(size_t)pid * args.n_theta + e] = R(0);
  } else {
    // ============ differential rollout + assembly (kernels.py:710-756) ============
    for (int t = 0; t < T; t++) {
      R xr[NX], ur[NU];
      load_z(t, xr, ur);
      if constexpr (!M::kLinearParams) M::template jac_vary<R>(th_r, dt_r, xr, ur, As, LDA, Bs);
      if (lane < NU) {
        const int r = lane;
        R s = ka[t * NU + r];
#pragma unroll
        for (int b = 0; b < NX; b++) s += Ka[(t * NU + r) * NX + b] * dXs[t * NX + b];
        dUs[t * NU + r] = s;
      }
      __syncwarp(gm);
      if (lane < NX) {
        const int a = lane;
        R s = R(0);
#pragma unroll
        for (int b = 0; b < NX; b++) s += As[a * LDA + b] * dXs[t * NX + b];
#pragma unroll
        for (int b = 0; b < NU; b++) s += Bs[a * NU + b] * dUs[t * NU + b];
        dXs[(t + 1) * NX + a] = s;
      }
      // assembly of stage t: dc = dz, dC = 0.5 (dz z' + z dz'), clamped rows/cols zero;
      // plus the optimal-cost terms sJ z and sJ/2 z z'
      auto zat = [&](int a) -> R { return a < NX ? Xs[t * NX + a] : Us[t * NU + a - NX]; };
      auto dzat = [&](int a) -> R { return a < NX ? dXs[t * NX + a] : dUs[t * NU + a - NX]; };
      auto clat = [&](int a) -> bool { return a >= NX && cl[t * NU + a - NX]; };
      if (dco) {
        for (int a = lane; a < NZ; a += G) {
          const R za = zat(a);
          dco[t * NZ + a] = (clat(a) ? R(0) : dzat(a)) + sJ * za;
        }
      }
      if (dCo) {
        if constexpr (DIAG) {
          for (int a = lane; a < NZ; a += G) {
            const R za = zat(a), da = dzat(a);
            const R v = clat(a) ? R(0) : R(0.5) * (da * za + za * da);
            dCo[t * NZ + a] = v + R(0.5) * sJ * za * za;
          }
        } else {
          for (int e = lane; e < NZ * NZ; e += G) {
            const int a = e / NZ, b = e % NZ;
            const R za = zat(a), zb = zat(b);
            const R v = (clat(a) || clat(b)) ? R(0) : R(0.5) * (dzat(a) * zb + za * dzat(b));
            dCo[(size_t)t * NZ * NZ + e] = v + R(0.5) * sJ * za * zb;
          }
        }
      }
      __syncwarp(gm);
    }

    // ============ co-state recursions: dtheta and the envelope terms (NEW) ========
    R gth[NTHL];
#pragma unroll
    for (int i = 0; i < NTHL; i++) gth[i] = R(0);
    constexpr int NZL = M::kLinearParams ? NZ : 1;
    R grow[NZL];  // linear model: row `lane` of [dA | dB]
#pragma unroll
    for (int i = 0; i < NZL; i++) grow[i] = R(0);
    if (want_adjoint) {
      for (int e = lane; e < NX; e += G) {
        lams[e] = R(0);
        lhs[e] = sXg ? sXg[T * NX + e] : R(0);
      }
      stage_C(T - 1, (T - 1) & 1);
      for (int t = T - 1; t >= 0; t--) {
        const int buf = t & 1;
        if (t > 0) {
          stage_C(t - 1, buf ^ 1);
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
          cp_async_wait_all();
        }
        R xr[NX], ur[NU];
        load_z(t, xr, ur);
        __syncwarp(gm);
        if constexpr (!M::kLinearParams) M::template jac_vary<R>(th_r, dt_r, xr, ur, As, LDA, Bs);
        __syncwarp(gm);
        if (want_theta) {
          if constexpr (M::kLinearParams) {
            if (lane < NX) {
              const int i = lane;
              const R lh = lhs[i], lm = lams[i], ls = sJ * lams[i];
#pragma unroll
              for (int j = 0; j < NX; j++) grow[j] += lh * xr[j] + lm * dXs[t * NX + j] + ls * xr[j];
#pragma unroll
              for (int j = 0; j < NU; j++) grow[NX + j] += lh * ur[j] + lm * dUs[t * NU + j] + ls * ur[j];
            }
          } else {
            R dx[NX], du[NU], lh[NX], lm[NX];
#pragma unroll
            for (int i = 0; i < NX; i++) {
              dx[i] = dXs[t * NX + i];
              lh[i] = lhs[i] + sJ * lams[i];
              lm[i] = lams[i];
            }
#pragma unroll
            for (int i = 0; i < NU; i++) du[i] = dUs[t * NU + i];
            M::template theta_grad<R>(th_r, dt_r, xr, ur, dx, du, lh, lm, gth);
          }
        }
        const R* Cs = Cb + buf * NCS;
        const R* cs = cb + buf * NZ;
        R nl = R(0), nh = R(0);
        if (lane < NX) {
          const int a = lane;
          R s1 = cg ? cs[a] : R(0);
          R s2 = sXg ? sXg[t * NX + a] : R(0);
          if constexpr (DIAG) {
            const R za = Xs[t * NX + a];
            s1 += Cs[a] * za;
            s2 += Cs[a] * dXs[t * NX + a];
          } else {
#pragma unroll
            for (int b = 0; b < NZ; b++) {
              const R zb = b < NX ? xr[b < NX ? b : 0] : ur[b >= NX ? b - NX : 0];
              const R db = b < NX ? dXs[t * NX + b] : dUs[t * NU + b - NX];
              s1 += Cs[a * NZ + b] * zb;
              s2 += Cs[a * NZ + b] * db;
            }
          }
#pragma unroll
          for (int b = 0; b < NX; b++) {
            s1 += As[b * LDA + a] * lams[b];
            s2 += As[b * LDA + a] * lhs[b];
          }
          nl = s1;
          nh = s2;
        }
        __syncwarp(gm);
        if (lane < NX) {
          lams[lane] = nl;
          lhs[lane] = nh;
        }
        __syncwarp(gm);
      }
      cp_async_wait_all();
      __syncwarp(gm);
    }
    if (args.dx0) {
      R* o = (R*)args.dx0 + (size_t)pid * NX;
      for (int e = lane; e < NX; e += G) o[e] = Vxs[e] + (want_adjoint ? sJ * lams[e] : R(0));
    }
    if (want_theta) {
      R* o = (R*)args.dtheta + (size_t)pid * args.n_theta;
      if constexpr (M::kLinearParams) {
        if (lane < NX) {
#pragma unroll
          for (int j = 0; j < NX; j++) o[lane * NX + j] = grow[j];
#pragma unroll
          for (int j = 0; j < NU; j++) o[NX * NX + lane * NU + j] = grow[NX + j];
        }
      } else {
        if (lane == 0)
          for (int i = 0; i < M::NTH; i++) o[i] = gth[i];
      }
    }
  }
  if (args.dX)
    for (int e = lane; e < (T + 1) * NX; e += G) ((R*)args.dX)[(size_t)pid * (T + 1) * NX + e] = dXs[e];
  if (args.dU)
    for (int e = lane; e < T * NU; e += G) ((R*)args.dU)[(size_t)pid * T * NU + e] = dUs[e];
  if (args.fail_t && lane == 0) args.fail_t[pid] = fail_t;
}

}  // namespace dmpc

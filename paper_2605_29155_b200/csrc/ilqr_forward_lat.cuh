// ilqr_forward_lat.cuh — latency-oriented forward iLQR: one 256-thread block per problem.
//
// Same algorithm and semantics as ilqr_forward_kernel (ilqr.py:154-247 over the range
// kernels of kernels.py), mapped for the smallest per-problem latency instead of the
// highest throughput (BASELINE config 2: B = 1 / 256 forward solves, "per-iter latency"):
//   * every n x n / m x n product of the Riccati stage is element-parallel (one thread per
//     output entry: 169 + 52 threads for MA / NB, Q_xx / Q_ux / Q_uu, N, V_xx), so a stage
//     is ~7 short phases separated by block barriers instead of one lane per row;
//   * the box QP on the control block runs on one thread while the block waits (the
//     n_u = 4 problem is a short serial chain);
//   * the line search runs one warp per step size (up to 8 candidates in one round): the
//     warp's lanes split the quadratic-cost rows and reduce with shuffles, and every
//     candidate writes its trajectory into its own buffer, so accepting any candidate is an
//     index swap (no re-roll);
//   * the problem's whole C / c (T stages) is staged into shared memory once.
// Precision follows the throughput kernel: Riccati algebra in R, trajectories / costs /
// feedforward in double, bound snapping of clamped feedforward coordinates.
#pragma once
#include "ilqr_forward.cuh"

namespace dmpc {

constexpr int kLatThreads = 256;

template <class M, bool DIAG, class R>
struct LatLayout {
  using D = Dims<M, DIAG, R>;
  int nbuf;
  int oPe, oX, oU, okg, oJc, oPr, oAs, oBs, oMA, oNB, oQxx, oQuxT, oQuu, oqu, oqx, oVx, oVxx, oN, oKT, oK, ozs,
      oL, oC, oc, oAT, oBT, ogz, obd, total;
  __host__ __device__ static LatLayout make(int T, int n_alpha) {
    LatLayout L;
    L.nbuf = 1 + n_alpha;
    int o = 0;
    auto take = [&](int bytes) { int r = o; o = align_up(o + bytes, 16); return r; };
    const int s = (int)sizeof(R);
    L.oPe = take(M::NP * 8);
    L.oX = take(L.nbuf * (T + 1) * D::XLD * 8);
    L.oU = take(L.nbuf * T * D::ULD * 8);
    L.okg = take(T * D::ULD * 8);
    L.oJc = take(16 * 8);  // candidate costs, dead flags, J, scalar state
    L.oPr = take(M::NP * s);
    L.oAs = take(D::NX * D::LDA * s);
    L.oBs = take(D::NX * D::LDB * s);
    L.oMA = take(D::NX * D::LDA * s);
    L.oNB = take(D::NX * D::LDB * s);
    L.oQxx = take(D::NX * D::LDA * s);
    L.oQuxT = take(D::NX * D::LDB * s);
    L.oQuu = take(D::NU * D::LDB * s);
    L.oqu = take(D::LDB * s);
    L.oqx = take(D::LDA * s);
    L.oVx = take(D::LDA * s);
    L.oVxx = take(D::NX * D::LDA * s);
    L.oN = take(D::NX * D::LDA * s);
    L.oKT = take(D::NX * D::LDB * s);
    L.oK = take(T * D::NU * D::LDA * s);
    L.ozs = take(D::ZLD * s);
    L.oL = take((D::NU * D::NU + 4 * D::NU + 8) * s);  // factor, inverses, du, flags
    L.oC = take(T * D::NCSP * s);
    L.oc = take(T * D::ZLD * s);
    // every stage's A_t, B_t and g_t = C_t z_t + c_t, evaluated in parallel before the sweep
    L.oAT = take(T * D::NX * D::LDA * s);
    L.oBT = take(T * D::NX * D::LDB * s);
    L.ogz = take(T * D::ZLD * s);
    L.obd = take(T * 2 * D::NU * 8);  // per stage: u_min - U_t, u_max - U_t (double)
    L.total = o;
    return L;
  }
};

// shared scalar state of the block's problem
struct LatState {
  double J;
  int active, fail_t, iterations, converged, diverged, nom, k_lo, ok, lam0, accept_best;
};

template <class M, bool DIAG, class R>
__global__ void __launch_bounds__(kLatThreads, 2) ilqr_forward_lat_kernel(const FwdArgs args) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  constexpr int LDA = D::LDA, LDB = D::LDB, ZLD = D::ZLD, XLD = D::XLD, ULD = D::ULD, NCSP = D::NCSP;
  using Lay = LatLayout<M, DIAG, R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ LatState st;
  __shared__ double Jc[8];
  __shared__ double Jw[8];  // per-warp partial candidate costs
  __shared__ int deadc[8];

  const int pid = blockIdx.x;
  if (pid >= args.B) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = args.T, NA = args.n_alpha;
  const Lay L = Lay::make(T, NA);
  unsigned char* base = smem_raw;
  double* P_e = (double*)(base + L.oPe);
  double* Xb = (double*)(base + L.oX);
  double* Ub = (double*)(base + L.oU);
  double* kg = (double*)(base + L.okg);
  R* P_r = (R*)(base + L.oPr);
  R* As = (R*)(base + L.oAs);
  R* Bs = (R*)(base + L.oBs);
  R* MA = (R*)(base + L.oMA);
  R* NB = (R*)(base + L.oNB);
  R* Qxx = (R*)(base + L.oQxx);
  R* QuxT = (R*)(base + L.oQuxT);
  R* Quu = (R*)(base + L.oQuu);
  R* qu = (R*)(base + L.oqu);
  R* qx = (R*)(base + L.oqx);
  R* Vx = (R*)(base + L.oVx);
  R* Vxx = (R*)(base + L.oVxx);
  R* Nn = (R*)(base + L.oN);
  R* KT = (R*)(base + L.oKT);
  R* Ks = (R*)(base + L.oK);
  R* zs = (R*)(base + L.ozs);
  R* Lf = (R*)(base + L.oL);  // [NU*NU] factor | [NU] inv | [NU] du | [NU] free | [NU] lo-hi scratch
  R* Cs = (R*)(base + L.oC);
  R* cs = (R*)(base + L.oc);
  R* AT = (R*)(base + L.oAT);  // [t][NX][LDA]
  R* BT = (R*)(base + L.oBT);  // [t][NX][LDB]
  R* gz = (R*)(base + L.ogz);  // [t][ZLD]
  double* bd = (double*)(base + L.obd);  // [t][lo(NU) | hi(NU)] bound offsets of the QP
  const int XB = (T + 1) * XLD, UB = T * ULD;  // buffer strides
  auto Xbuf = [&](int b) { return Xb + b * XB; };
  auto Ubuf = [&](int b) { return Ub + b * UB; };

  // ---- parameters, constant Jacobian structure, cost tensors, x0 / U_warm ----
  const R* thg = (const R*)args.theta + (size_t)args.theta_stride * pid;
  if constexpr (!M::kLinearParams) {
    if (tid == 0) {
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
  }
  __syncthreads();
  const double dt_e = args.dt;
  const R dt_r = (R)args.dt;
  if constexpr (M::kLinearParams) {
    for (int e = tid; e < NX * NX; e += kLatThreads) As[(e / NX) * LDA + e % NX] = thg[e];
    for (int e = tid; e < NX * NU; e += kLatThreads) Bs[(e / NU) * LDB + e % NU] = thg[NX * NX + e];
  } else if (warp == 0) {
    // one warp: jac_const zero-fills and then lets lane 0 write the constant entries, which is
    // ordered only within a warp (a block-wide fill could land after lane 0's writes)
    M::template jac_const<R>(P_r, dt_r, As, LDA, Bs, LDB, lane, 32);
  }
  {
    const R* Cg = (const R*)args.C + (size_t)pid * T * D::NCS;
    const R* cg = (const R*)args.c + (size_t)pid * T * NZ;
    if constexpr (DIAG) {
      for (int e = tid; e < T * NZ; e += kLatThreads) Cs[(e / NZ) * NCSP + e % NZ] = Cg[e];
    } else {
      for (int e = tid; e < T * NZ * NZ; e += kLatThreads) {
        const int t = e / (NZ * NZ), r = e % (NZ * NZ);
        Cs[t * NCSP + (r / NZ) * ZLD + r % NZ] = Cg[e];
      }
    }
    for (int e = tid; e < T * NZ; e += kLatThreads) cs[(e / NZ) * ZLD + e % NZ] = cg[e];
    const R* xg = (const R*)args.x0 + (size_t)pid * NX;
    for (int e = tid; e < NX; e += kLatThreads) Xbuf(0)[e] = (double)xg[e];
    const R* ug = (const R*)args.U_warm + (size_t)pid * T * NU;
    for (int e = tid; e < T * NU; e += kLatThreads) {
      double v = (double)ug[e];
      const int r = e % NU;
      const double lo = args.u_min[r], hi = args.u_max[r];
      v = v < lo ? lo : v;  // np.clip (ilqr.py:165)
      v = v > hi ? hi : v;
      Ubuf(0)[(e / NU) * ULD + r] = v;
      kg[(e / NU) * ULD + r] = 0.0;
    }
  }
  __syncthreads();  // As / Bs (constant structure) complete
  for (int e = tid; e < T * NX * LDA; e += kLatThreads) AT[e] = As[e % (NX * LDA)];
  for (int e = tid; e < T * NX * LDB; e += kLatThreads) BT[e] = Bs[e % (NX * LDB)];
  R* Ko = args.K ? (R*)args.K + (size_t)pid * T * NU * NX : nullptr;
  R* ahist = args.alpha_hist ? (R*)args.alpha_hist + (size_t)pid * args.K_max : nullptr;
  R* jhist = args.J_hist ? (R*)args.J_hist + (size_t)pid * (args.K_max + 1) : nullptr;
  if (ahist)
    for (int e = tid; e < args.K_max; e += kLatThreads) ahist[e] = R(0);
  if (tid == 0) {
    st.J = 0.0;
    st.active = 1;
    st.fail_t = -1;
    st.iterations = 0;
    st.converged = 0;
    st.diverged = 0;
    st.nom = 0;
    st.k_lo = T;
  }
  __syncthreads();

  // warp-level stage cost 0.5 z'Cz + c'z in double (kernels.py:133-145): lane i < NZ owns
  // row i; the warp reduces. Every lane returns the identical total.
  auto warp_cost = [&](const R* C_t, const R* c_t, const double (&x)[NX], const double (&u)[NU]) -> double {
    double z[NZ];
#pragma unroll
    for (int i = 0; i < NX; i++) z[i] = x[i];
#pragma unroll
    for (int i = 0; i < NU; i++) z[NX + i] = u[i];
    double zi = 0.0;
#pragma unroll
    for (int k = 0; k < NZ; k++)
      if (lane == k) zi = z[k];
    double part = 0.0;
    if (lane < NZ) {
      if constexpr (DIAG) {
        part = 0.5 * zi * ((double)C_t[lane] * zi) + (double)c_t[lane] * zi;
      } else {
        R crow[NZ];
        lds_row<NZ>(C_t + lane * ZLD, crow);
        double ra[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NZ; j++) ra[j & 3] += (double)crow[j] * z[j];
        const double row = (ra[0] + ra[1]) + (ra[2] + ra[3]);
        part = 0.5 * zi * row + (double)c_t[lane] * zi;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    return part;
  };


  // =========================== initial rollout (kernels.py:161-178), warp 0 =========
  if (warp == 0) {
    double x[NX];
    lds_row_d<NX>(Xbuf(0), x);
    double J = 0.0;
    int fail = -1;
    for (int t = 0; t < T; t++) {
      double u[NU];
      lds_row_d<NU>(Ubuf(0) + t * ULD, u);
      J += warp_cost(Cs + t * NCSP, cs + t * ZLD, x, u);
      double xn[NX];
      step_e<M, R>(P_e, dt_e, As, LDA, Bs, LDB, x, u, xn);
      bool fin = true;
#pragma unroll
      for (int i = 0; i < NX; i++) {
        fin &= finite_(xn[i]);
        x[i] = xn[i];
        if (lane == i) Xbuf(0)[(t + 1) * XLD + i] = xn[i];
      }
      if (!fin) {
        fail = t;
        // rows past the failure keep the reference Workspace's zero init (ilqr.py:84-133)
        for (int e = lane; e < (T - 1 - t) * XLD; e += 32) Xbuf(0)[(t + 2) * XLD + e] = 0.0;
        break;
      }
    }
    if (lane == 0) {
      if (fail >= 0) {  // rollout_failed (ilqr.py:196-200)
        st.fail_t = fail;
        st.active = 0;
        st.J = INFINITY;
        st.diverged = 1;
      } else {
        st.J = J;
      }
      if (jhist) jhist[0] = (R)st.J;
    }
  }
  __syncthreads();

#ifdef DMPC_LAT_PROF
  __shared__ long long prof[16];
  if (tid < 16) prof[tid] = 0;
  __syncthreads();
  long long tp = clock64();
#define LAT_MARK(k)                          \
  if (tid == 0) {                            \
    const long long n_ = clock64();          \
    prof[k] += n_ - tp;                      \
    tp = n_;                                 \
  }
#else
#define LAT_MARK(k)
#endif
  // =============================== iterations ==================================
  int it = 0;
  for (; it < args.K_max && st.active; it++) {
    const int nom = st.nom;
    double* Xn = Xbuf(nom);
    double* Un = Ubuf(nom);
    // V = 0 (ilqr.py:208-209)
    for (int e = tid; e < NX * LDA; e += kLatThreads) Vxx[e] = R(0);
    for (int e = tid; e < LDA; e += kLatThreads) Vx[e] = R(0);
    __syncthreads();
    // Stage-parallel prologue: every stage's Jacobians (thread t < T: the state-dependent
    // entries of A_t, B_t at the nominal) and cost gradient g_t = C_t z_t + c_t (one thread
    // per entry), so the sequential stages below carry only the Riccati recursion.
    if constexpr (!M::kLinearParams) {
      for (int t = tid; t < T; t += kLatThreads) {
        R xr[NX], ur[NU];
#pragma unroll
        for (int i = 0; i < NX; i++) xr[i] = (R)Xn[t * XLD + i];
#pragma unroll
        for (int i = 0; i < NU; i++) ur[i] = (R)Un[t * ULD + i];
        M::template jac_vary<R>(P_r, dt_r, xr, ur, AT + t * NX * LDA, LDA, BT + t * NX * LDB, LDB);
      }
    }
    for (int e = tid; e < T * NZ; e += kLatThreads) {
      const int t = e / NZ, a = e - (e / NZ) * NZ;
      const R* C_t = Cs + t * NCSP;
      R s0 = cs[t * ZLD + a], s1 = R(0);
      if constexpr (DIAG) {
        s0 += C_t[a] * (R)(a < NX ? Xn[t * XLD + a] : Un[t * ULD + a - NX]);
      } else {
#pragma unroll
        for (int j = 0; j < NZ; j++) {
          const R p = C_t[a * ZLD + j] * (R)(j < NX ? Xn[t * XLD + j] : Un[t * ULD + j - NX]);
          if (j & 1) s1 += p; else s0 += p;
        }
      }
      gz[t * ZLD + a] = s0 + s1;
    }
    for (int e = tid; e < T * NU; e += kLatThreads) {
      const int t = e / NU, i = e - (e / NU) * NU;
      bd[t * 2 * NU + i] = args.u_min[i] - Un[t * ULD + i];
      bd[t * 2 * NU + NU + i] = args.u_max[i] - Un[t * ULD + i];
    }
    __syncthreads();
    LAT_MARK(1);
    bool failed_sweep = false;
    for (int t = T - 1; t >= 0; t--) {
      const R* C_t = Cs + t * NCSP;
      const R* At = AT + t * NX * LDA;
      const R* Bt = BT + t * NX * LDB;
      // P2: MA = Vxx A, NB = Vxx B, qx = g_x + A'Vx, qu = g_u + B'Vx  (kernels.py:395-421)
      if (tid < NX * NX) {
        const int a = tid / NX, b = tid % NX;
        R s0 = R(0), s1 = R(0);
#pragma unroll
        for (int r = 0; r < NX; r++) {
          const R p = Vxx[a * LDA + r] * At[r * LDA + b];
          if (r & 1) s1 += p; else s0 += p;
        }
        MA[a * LDA + b] = s0 + s1;
      } else if (tid < NX * NX + NX * NU) {
        const int e = tid - NX * NX, a = e / NU, i = e % NU;
        R s = R(0);
#pragma unroll
        for (int r = 0; r < NX; r++) s += Vxx[a * LDA + r] * Bt[r * LDB + i];
        NB[a * LDB + i] = s;
      } else if (tid < NX * NX + NX * NU + NZ) {
        const int a = tid - NX * NX - NX * NU;
        const R s0 = gz[t * ZLD + a];
        R s1 = R(0);
        if (a < NX) {
#pragma unroll
          for (int r = 0; r < NX; r++) s1 += At[r * LDA + a] * Vx[r];
          qx[a] = s0 + s1;
        } else {
#pragma unroll
          for (int r = 0; r < NX; r++) s1 += Bt[r * LDB + (a - NX)] * Vx[r];
          qu[a - NX] = s0 + s1;
        }
      }
      __syncthreads();
      LAT_MARK(2);
      // P3: Qxx = Cxx + A'MA, Qux = Cux + B'MA, Quu = Cuu + B'NB  (kernels.py:422-439)
      if (tid < NX * NX) {
        const int a = tid / NX, b = tid % NX;
        R s0, s1 = R(0);
        if constexpr (DIAG) s0 = (a == b) ? C_t[a] : R(0);
        else s0 = C_t[a * ZLD + b];
#pragma unroll
        for (int r = 0; r < NX; r++) {
          const R p = At[r * LDA + a] * MA[r * LDA + b];
          if (r & 1) s1 += p; else s0 += p;
        }
        Qxx[a * LDA + b] = s0 + s1;
      } else if (tid < NX * NX + NX * NU) {
        const int e = tid - NX * NX, b = e / NU, i = e % NU;
        R s;
        if constexpr (DIAG) s = R(0);
        else s = C_t[(NX + i) * ZLD + b];
#pragma unroll
        for (int r = 0; r < NX; r++) s += Bt[r * LDB + i] * MA[r * LDA + b];
        QuxT[b * LDB + i] = s;
      } else if (tid < NX * NX + NX * NU + NU * NU) {
        const int e = tid - NX * NX - NX * NU, i = e / NU, j = e % NU;
        R s;
        if constexpr (DIAG) s = (i == j) ? C_t[NX + i] : R(0);
        else s = C_t[(NX + i) * ZLD + NX + j];
#pragma unroll
        for (int r = 0; r < NX; r++) s += Bt[r * LDB + i] * NB[r * LDB + j];
        Quu[i * LDB + j] = s;
      }
      __syncthreads();
      LAT_MARK(3);
      // P4: the lambda-regularised box QP on the control block (kernels.py:440-489), run
      // redundantly by the NX lanes that then form one K column each and the V_x update
      // (kernels.py:481-498): one phase, the factor stays in registers.
      if (tid < NX) {
        const int b = tid;
        R quu[NU][NU], qv[NU], lo[NU], hi[NU], du[NU];
        bool fr[NU], lam0 = true;
        Chol<NU, R> ch;
        double lod[NU], hid[NU];
#pragma unroll
        for (int i = 0; i < NU; i++) {
#pragma unroll
          for (int j = 0; j < NU; j++) quu[i][j] = Quu[i * LDB + j];
          qv[i] = qu[i];
          lod[i] = bd[t * 2 * NU + i];
          hid[i] = bd[t * 2 * NU + NU + i];
          lo[i] = (R)lod[i];
          hi[i] = (R)hid[i];
        }
        // straight-line interior fast path; the full lambda / projected-Newton solve only
        // when it does not apply (the box binds, or Quu is not positive definite)
        bool ok = qp_interior<NU, R>(quu, qv, lo, hi, (R)args.boxqp_tol, du, fr, ch);
        if (!ok) ok = stage_qp<NU, R>(quu, qv, lo, hi, args.boxqp_max_iter, (R)args.boxqp_tol, du, fr, ch, lam0);
        if (b == 0) {
          st.ok = ok;
          st.lam0 = lam0;
          if (ok) {
#pragma unroll
            for (int i = 0; i < NU; i++) {
              double kd = (double)du[i];  // bound snapping (see ilqr_forward_kernel)
              if (du[i] <= lo[i]) kd = lod[i];
              else if (du[i] >= hi[i]) kd = hid[i];
              kg[t * ULD + i] = kd;
            }
          } else {
            st.fail_t = t;
            st.active = 0;
          }
        }
        if (ok) {
          R quxc[NU], rhs[NU], sol[NU], kcol[NU];
#pragma unroll
          for (int i = 0; i < NU; i++) {
            quxc[i] = QuxT[b * LDB + i];
            rhs[i] = fr[i] ? quxc[i] : R(0);
          }
          chol_solve<NU, R>(ch, rhs, sol);
#pragma unroll
          for (int i = 0; i < NU; i++) {
            kcol[i] = fr[i] ? -sol[i] : R(0);
            KT[b * LDB + i] = kcol[i];
            Ks[(t * NU + i) * LDA + b] = kcol[i];
            if (Ko) Ko[(t * NU + i) * NX + b] = kcol[i];
          }
          R sv = qx[b];
#pragma unroll
          for (int r = 0; r < NU; r++) {
            R rowq = R(0);
#pragma unroll
            for (int q = 0; q < NU; q++) rowq += quu[r][q] * du[q];
            sv += kcol[r] * (rowq + qv[r]) + quxc[r] * du[r];
          }
          Vx[b] = sv;
        }
      }
      __syncthreads();
      LAT_MARK(4);
      if (!st.ok) {
        failed_sweep = true;
        break;
      }
      const bool lam0 = st.lam0 != 0;
      // P5: V_xx = (N + N')/2 with N = Qxx + Qux'K (lean) or the full value update
      // (kernels.py:499-512); thread (a, b) forms both N[a,b] and N[b,a] (no extra phase)
      if (tid < NX * NX) {
        const int a = tid / NX, b = tid % NX;
        auto nval = [&](int i, int j) -> R {
          R s = Qxx[i * LDA + j];
          if (lam0) {
#pragma unroll
            for (int r = 0; r < NU; r++) s += QuxT[i * LDB + r] * KT[j * LDB + r];
          } else {
#pragma unroll
            for (int r = 0; r < NU; r++) {
              R kq = R(0);
#pragma unroll
              for (int q = 0; q < NU; q++) kq += Quu[r * LDB + q] * KT[j * LDB + q];
              s += (KT[i * LDB + r] * kq + KT[i * LDB + r] * QuxT[j * LDB + r]) + QuxT[i * LDB + r] * KT[j * LDB + r];
            }
          }
          return s;
        };
        Vxx[a * LDA + b] = R(0.5) * (nval(a, b) + nval(b, a));
      }
      if (tid == 0) st.k_lo = t;
      __syncthreads();
      LAT_MARK(5);
    }
    (void)failed_sweep;
    LAT_MARK(7);

    // --------------------- line search: one warp per step size -------------------
    // Phase A: warp a rolls candidate a out (feedback law + dynamics only, the chain that
    // is inherently sequential in t) into its own trajectory buffer. Phase B: all 8 warps
    // evaluate every candidate's stage costs in parallel and reduce them (the costs are off
    // the state recursion, so they no longer sit on its critical path).
    const int act = st.active;
    if (act && warp < NA) {
      const int a = warp;
      const double alpha = args.alphas[a];
      const int cb = (nom + 1 + a) % L.nbuf;  // candidate buffer (never the nominal)
      double* Xc = Xbuf(cb);
      double* Uc = Ubuf(cb);
      double x[NX];
      lds_row_d<NX>(Xn, x);
      bool dm = false;
      for (int t = 0; t < T; t++) {
        // nominal row, controls, gains: independent of the candidate state
        double xbar[NX];
        lds_row_d<NX>(Xn + t * XLD, xbar);
        const int r = lane < NU ? lane : 0;
        double v = Un[t * ULD + r] + alpha * kg[t * ULD + r];
        R krow[NX];
        lds_row<NX>(Ks + (t * NU + r) * LDA, krow);
        v = feedback<NX>(v, krow, x, xbar);
        const double lo = args.u_min[r], hi = args.u_max[r];
        if (v < lo) v = lo;
        else if (v > hi) v = hi;
        double u[NU];
#pragma unroll
        for (int q = 0; q < NU; q++) u[q] = __shfl_sync(0xffffffffu, v, q);
        double xn[NX];
        step_e<M, R>(P_e, dt_e, As, LDA, Bs, LDB, x, u, xn);
        if (lane < NU) Uc[t * ULD + lane] = v;
        double xl = x[0];  // lane i stores x_i: a select chain and one store
#pragma unroll
        for (int i = 1; i < NX; i++) xl = lane == i ? x[i] : xl;
        if (lane < NX) Xc[t * XLD + lane] = xl;
#pragma unroll
        for (int i = 0; i < NX; i++) x[i] = xn[i];
      }
      // Dead candidates (kernels.py:569-574): a non-finite x_{t+1} for t < T-1 makes the
      // stage-(t+1) cost non-finite (z_i * (C z)_i with z_i = inf / nan), which phase B
      // detects; x_T has no stage cost and is checked here. So the per-stage finiteness
      // tests of the reference are decided exactly, off the rollout's critical path.
      double xl = x[0];
#pragma unroll
      for (int i = 1; i < NX; i++) xl = lane == i ? x[i] : xl;
      if (lane < NX) Xc[T * XLD + lane] = xl;
#pragma unroll
      for (int i = 0; i < NX; i++) dm |= !finite_(x[i]);
      if (lane == 0) deadc[a] = dm;
    }
    __syncthreads();
    LAT_MARK(8);
    if (act) {
      // Phase B: (candidate, stage, row) items; WPC warps per candidate share its T * NZ rows
      const int wpc = 8 / NA;  // NA <= 8
      const int a = warp / wpc;
      double part = 0.0;
      if (a < NA) {
        const int cb = (nom + 1 + a) % L.nbuf;
        const double* Xc = Xbuf(cb);
        const double* Uc = Ubuf(cb);
        const int P = wpc * 32, s0 = (warp - a * wpc) * 32 + lane;
        for (int e = s0; e < T * NZ; e += P) {
          const int t = e / NZ, i = e - (e / NZ) * NZ;
          double x[NX], u[NU];
          lds_row_d<NX>(Xc + t * XLD, x);
          lds_row_d<NU>(Uc + t * ULD, u);
          const R* C_t = Cs + t * NCSP;
          const R* c_t = cs + t * ZLD;
          const double zi = i < NX ? Xc[t * XLD + i] : Uc[t * ULD + i - NX];
          if constexpr (DIAG) {
            part += 0.5 * zi * ((double)C_t[i] * zi) + (double)c_t[i] * zi;
          } else {
            R crow[NZ];
            lds_row<NZ>(C_t + i * ZLD, crow);
            double ra[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int j = 0; j < NX; j++) ra[j & 3] += (double)crow[j] * x[j];
#pragma unroll
            for (int j = 0; j < NU; j++) ra[(NX + j) & 3] += (double)crow[NX + j] * u[j];
            part += 0.5 * zi * ((ra[0] + ra[1]) + (ra[2] + ra[3])) + (double)c_t[i] * zi;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
        if (lane == 0) Jw[warp] = part;
      }
      __syncthreads();
      if (tid < NA) {  // fixed-order sum of the candidate's warp partials (repeatable); a
                       // non-finite state or stage cost makes the candidate dead
        double J = 0.0;
        for (int w = 0; w < wpc; w++) J += Jw[tid * wpc + w];
        const bool dm = deadc[tid] != 0 || !finite_(J);
        deadc[tid] = dm;
        Jc[tid] = dm ? INFINITY : J;
      }
    }
    __syncthreads();
    LAT_MARK(6);
    // ------------------------- epilogue (ilqr.py:216-244) -----------------------
    if (tid == 0) {
      if (act) st.iterations = it + 1;
      int best = 0;
      double best_J = act ? Jc[0] : 0.0;
      bool alld = act ? deadc[0] != 0 : false;
      for (int a = 1; a < NA && act; a++) {
        if (Jc[a] < best_J) {
          best_J = Jc[a];
          best = a;
        }
        alld = alld && deadc[a] != 0;
      }
      const bool all_dead = act && alld;
      const bool accept = act && !all_dead && (best_J < st.J);
      if (ahist) ahist[it] = accept ? (R)args.alphas[best] : R(0);
      const double J_prev = st.J;
      if (accept) {
        st.J = best_J;
        st.nom = (nom + 1 + best) % L.nbuf;
      }
      if (all_dead) {
        st.diverged = 1;
        st.active = 0;
      }
      const double rel = fabs(J_prev - st.J) / fmax(1.0, fabs(J_prev));
      const bool no_step = act && !all_dead && !accept;
      if ((act && !all_dead) && (no_step || rel <= args.conv_tol)) {
        st.converged = 1;
        st.active = 0;
      }
      if (jhist) jhist[it + 1] = (R)st.J;
    }
    __syncthreads();
  }

#ifdef DMPC_LAT_PROF
  if (tid == 0 && pid == 0)
    printf("lat prof cycles: prologue %lld P2 %lld P3 %lld P4(QP+K) %lld P5(V) %lld sweep-end %lld "
           "LS-rollout %lld LS-costs %lld\n", prof[1], prof[2], prof[3], prof[4], prof[5], prof[7], prof[8], prof[6]);
#endif
  // ================================ outputs ====================================
  if (jhist && tid == 0)
    for (int e = it + 1; e <= args.K_max; e++) jhist[e] = (R)st.J;
  const double* Xn = Xbuf(st.nom);
  const double* Un = Ubuf(st.nom);
  const bool failed = st.fail_t >= 0 || st.diverged;
  R* Xo = (R*)args.X + (size_t)pid * (T + 1) * NX;
  for (int e = tid; e < (T + 1) * NX; e += kLatThreads) Xo[e] = (R)Xn[(e / NX) * XLD + e % NX];
  R* Uo = (R*)args.U + (size_t)pid * T * NU;
  for (int e = tid; e < T * NU; e += kLatThreads) Uo[e] = (R)Un[(e / NU) * ULD + e % NU];
  if (args.clamped) {
    uint8_t* co = args.clamped + (size_t)pid * T * NU;
    for (int e = tid; e < T * NU; e += kLatThreads) {
      const int r = e % NU;
      const double v = Un[(e / NU) * ULD + r];
      co[e] = (uint8_t)(v <= args.u_min[r] || v >= args.u_max[r]);
    }
  }
  if (Ko && st.k_lo > 0)
    for (int e = tid; e < st.k_lo * NU * NX; e += kLatThreads) Ko[e] = R(0);
  if (args.k) {
    R* ko = (R*)args.k + (size_t)pid * T * NU;
    for (int e = tid; e < T * NU; e += kLatThreads) ko[e] = (R)kg[(e / NU) * ULD + e % NU];
  }
  if (tid == 0) {
    ((R*)args.J)[pid] = (R)st.J;
    if (args.iters) args.iters[pid] = st.iterations;
    if (args.converged) args.converged[pid] = (uint8_t)(st.converged && !failed);
    if (args.diverged) args.diverged[pid] = (uint8_t)st.diverged;
    if (args.fail_t) args.fail_t[pid] = st.fail_t;
  }
}

}  // namespace dmpc

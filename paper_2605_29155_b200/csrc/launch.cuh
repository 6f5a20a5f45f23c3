// launch.cuh — host-side launch planning for the DiffMPC kernels (shared by the
// per-model instantiation units inst_*.cu and the C ABI in capi.cu).
#pragma once
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/diffmpc.h"
#include "ilqr_backward.cuh"
#include "ilqr_forward_lat.cuh"

namespace dmpc {

int fail(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
extern std::atomic<int64_t> g_launches;
int max_smem_optin();
// the library's stream-ordered pool for internal workspaces (current device; memory is kept
// cached across calls instead of going back to the driver at every synchronisation)
cudaMemPool_t work_pool();

// default lanes per problem (a lane owns ceil(n_x / G) state rows)
constexpr int default_group(int nx) { return nx <= 4 ? 4 : (nx <= 8 ? 8 : 16); }
int group_env();  // DIFFMPC_GROUP override (0 = none), read once


template <class M>
int check_theta(const DiffMPCProblem* p) {
  if (p->n_theta != M::NTH) return fail("model kind %d expects %d parameters, got %d", M::KIND, M::NTH, p->n_theta);
  return 0;
}

// Problems per block: among gpb in {128/G, 64/G, 32/G, ...} pick the one that keeps the
// most problems resident per SM (occupancy API: registers + shared memory).
template <class Lay, class K>
int plan(K kern, int B, int T, int G, int& gpb, int& stride, int* per_sm = nullptr, int bytes = 0) {
  const Lay L = Lay::make(T);
  // per-group stride = whole 128-byte lines + G banks: the 32/G groups of a warp start G
  // banks apart, so a warp-wide access of consecutive elements (lane = row or column
  // index, one per group) covers all 32 banks instead of hitting the same 16 twice
  // (`bytes` > 0: the group's block size when it differs from Lay::make(T).total)
  stride = bytes > 0 ? (bytes + 127) / 128 * 128 + 4 * G : group_stride<Lay>(T, G);
  (void)L;
  const int limit = max_smem_optin();
  int best = -1, best_res = -1;
  for (int g = 128 / G; g >= 1; g /= 2) {
    const int smem = g * stride;
    if (smem > limit) continue;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, g * G, smem) != cudaSuccess) nb = 1;
    const int res = nb * g;
    if (res > best_res) {
      best_res = res;
      best = g;
      if (per_sm) *per_sm = nb;
    }
  }
  cudaGetLastError();
  if (best < 0)
    return fail("horizon T=%d needs %d bytes of shared memory per problem (limit %d)", T, stride, limit);
  gpb = best;
  if (B < gpb) gpb = B > 0 ? B : 1;
  return 0;
}

int num_sms();

// Forward workspace: [work counter (256 B)] [gains K (B, T, NU, LDA) of R]
//                    [packed cost records (B, T, REC) of R]
inline size_t rup128(size_t v) { return (v + 127) / 128 * 128; }
// per-problem strides (bytes), 128-byte multiples: no L2 line is shared by two problems
inline size_t fwd_gain_stride(int T, int nx, int nu, int elem) {
  const int vn = 16 / elem;
  const size_t lda = (size_t)((nx + vn - 1) / vn * vn);
  return rup128((size_t)T * nu * lda * elem);
}
inline size_t fwd_rec_elems(int nx, int nu, int elem, bool diag) {
  const int vn = 16 / elem, nz = nx + nu;
  const size_t zld = (size_t)((nz + vn - 1) / vn * vn);
  return (diag ? zld : nz * zld) + zld;
}
inline size_t fwd_rec_stride(int T, int nx, int nu, int elem, bool diag) {
  return rup128((size_t)T * fwd_rec_elems(nx, nu, elem, diag) * elem);
}
inline size_t fwd_workspace_bytes(int B, int T, int nx, int nu, int elem, bool diag) {
  return 256 + (size_t)B * (fwd_gain_stride(T, nx, nu, elem) + fwd_rec_stride(T, nx, nu, elem, diag));
}

template <class M, int G, bool DIAG, class R>
int fwd_impl(const DiffMPCProblem* p, const DiffMPCForwardIO* io, cudaStream_t s) {
  if (check_theta<M>(p)) return -1;
  if (!io) return fail("forward: null io");
  if (p->B == 0) return 0;  // empty batch: nothing to launch (empty arrays may be NULL)
  if (!io->X || !io->U || !io->J || !io->C || !io->c || !io->x0 || !io->U_warm || (M::NTH > 0 && !io->theta))
    return fail("forward: required pointer is NULL");
  FwdArgs a;
  memset(&a, 0, sizeof a);
  a.B = p->B; a.T = p->T; a.K_max = p->K_max; a.n_alpha = p->n_alpha;
  a.boxqp_max_iter = p->boxqp_max_iter; a.theta_stride = p->theta_stride;
  a.dt = p->dt; a.conv_tol = p->conv_tol; a.boxqp_tol = p->boxqp_tol;
  for (int i = 0; i < 8; i++) {
    a.u_min[i] = p->u_min[i]; a.u_max[i] = p->u_max[i]; a.alphas[i] = p->alphas[i];
  }
  a.theta = io->theta; a.C = io->C; a.c = io->c; a.x0 = io->x0; a.U_warm = io->U_warm;
  a.X = io->X; a.U = io->U; a.J = io->J; a.K = io->K; a.k = io->k; a.iters = io->iters;
  a.converged = io->converged; a.diverged = io->diverged; a.fail_t = io->fail_t;
  a.clamped = io->clamped; a.alpha_hist = io->alpha_hist; a.J_hist = io->J_hist;
  // Small batches take the latency-oriented kernel (one block per problem) while the
  // grid cannot fill the GPU with the throughput mapping; DIFFMPC_FWD=lat|tput forces one.
  {
    static int mode = -1, lat_max = 0;
    if (mode < 0) {
      const char* e = getenv("DIFFMPC_FWD");
      mode = (e && std::string(e) == "lat") ? 1 : ((e && std::string(e) == "tput") ? 2 : 0);
      const char* m = getenv("DIFFMPC_LAT_MAX");
      lat_max = m ? atoi(m) : 2 * num_sms();
    }
    const LatLayout<M, DIAG, R> LL = LatLayout<M, DIAG, R>::make(p->T, p->n_alpha);
    const bool fits = LL.total <= max_smem_optin() - 1024;
    // per-call choice (kernel_select) wins; DIFFMPC_FWD only steers the auto choice
    const int sel = p->kernel_select != DIFFMPC_KERNEL_AUTO ? p->kernel_select : (mode == 1 ? 2 : (mode == 2 ? 1 : 0));
    if (fits && (sel == DIFFMPC_KERNEL_LATENCY || (sel == DIFFMPC_KERNEL_AUTO && p->B <= lat_max))) {
      auto lk = ilqr_forward_lat_kernel<M, DIAG, R>;
      if (LL.total > 48 * 1024) cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, LL.total);
      lk<<<p->B, kLatThreads, LL.total, s>>>(a);
      g_launches.fetch_add(1);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return fail("forward (latency) launch failed: %s", cudaGetErrorString(e));
      return 0;
    }
  }
  // warp lockstep of the groups (ilqr_forward_kernel): auto = fixed-work solves (conv_tol <= 0:
  // every problem runs ~K_max iterations) and long horizons (T >= 16: wider spread of
  // iteration counts; B=65536 hover batch, T=20: 20.7 vs 26.5 ms, T=40: 50.2 vs 66.0 ms;
  // T=10: 5.45 vs 5.26 ms); DIFFMPC_LOCKSTEP=0|1 forces it
  static int ls_env = -2;
  if (ls_env == -2) {
    const char* e = getenv("DIFFMPC_LOCKSTEP");
    ls_env = e ? (atoi(e) != 0) : -1;
  }
  const bool lock = ls_env >= 0 ? ls_env != 0 : (p->conv_tol <= 0.0 || p->T >= 16);
  auto kern = lock ? ilqr_forward_kernel<M, G, DIAG, R, true> : ilqr_forward_kernel<M, G, DIAG, R, false>;
  if constexpr (sizeof(R) == 4) {  // the bench horizon with compile-time shared-memory offsets
    if (p->T == 10) kern = lock ? ilqr_forward_kernel<M, G, DIAG, R, true, 10> : ilqr_forward_kernel<M, G, DIAG, R, false, 10>;
    if constexpr (std::is_same_v<M, Quad13>) {  // the config-5 sweep horizons of the BASELINE model
      if (p->T == 5 && !lock) kern = ilqr_forward_kernel<M, G, DIAG, R, false, 5>;
      if (p->T == 20 && lock) kern = ilqr_forward_kernel<M, G, DIAG, R, true, 20>;
      if (p->T == 40 && lock) kern = ilqr_forward_kernel<M, G, DIAG, R, true, 40>;
    }
  }
  int per_sm = 1;
  if ((lock ? plan<FwdLayout<M, DIAG, R, true>>(kern, p->B, p->T, G, a.gpb, a.smem_stride, &per_sm)
            : plan<FwdLayout<M, DIAG, R, false>>(kern, p->B, p->T, G, a.gpb, a.smem_stride, &per_sm)))
    return -1;
  if (const char* e = getenv("DIFFMPC_GPB")) {  // tuning override (even, keeps warps full)
    const int g = atoi(e);
    if (g >= 2 && g % 2 == 0 && g * G <= 128 && g * a.smem_stride <= max_smem_optin()) {  // launch bounds: 128 threads
      a.gpb = g;
      const int smem_g = g * a.smem_stride;
      if (smem_g > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_g);
      int nb = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, g * G, smem_g) == cudaSuccess && nb > 0) per_sm = nb;
    }
  }
  if (p->B < a.gpb) {  // small batch: one block of the next power of two >= B groups
    int g = 1;
    while (g < p->B) g *= 2;
    a.gpb = g;
  }
  const int smem = a.gpb * a.smem_stride;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // persistent grid: at most the resident blocks; groups claim problems dynamically
  const int need_blocks = (p->B + a.gpb - 1) / a.gpb;
  const int resident = per_sm * num_sms();
  const int blocks = need_blocks < resident ? need_blocks : resident;
  // workspace (caller-provided, else stream-ordered pool allocation)
  const size_t wsb = fwd_workspace_bytes(p->B, p->T, M::NX, M::NU, (int)sizeof(R), DIAG);
  void* ws = io->workspace;
  bool own = false;
  if (!ws || io->workspace_bytes < wsb) {
    if (cudaMallocFromPoolAsync(&ws, wsb, work_pool(), s) != cudaSuccess)
      return fail("forward: workspace allocation of %zu bytes failed", wsb);
    own = true;
  }
  const size_t gs = fwd_gain_stride(p->T, M::NX, M::NU, (int)sizeof(R));
  const size_t ps = fwd_rec_stride(p->T, M::NX, M::NU, (int)sizeof(R), DIAG);
  a.ctr = (int*)ws;
  a.Kw = (unsigned char*)ws + 256;
  a.Pw = (unsigned char*)ws + 256 + (size_t)p->B * gs;
  a.kw_stride = (long long)(gs / sizeof(R));
  a.pw_stride = (long long)(ps / sizeof(R));
  cudaMemsetAsync(ws, 0, sizeof(int), s);
  kern<<<blocks, a.gpb * G, smem, s>>>(a);
  g_launches.fetch_add(1);
  cudaError_t e = cudaGetLastError();
  if (own) cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return fail("forward launch failed: %s", cudaGetErrorString(e));
  return 0;
}

template <class M, int G, bool DIAG, class R>
int bwd_impl(const DiffMPCProblem* p, const DiffMPCBackwardIO* io, cudaStream_t s) {
  if (check_theta<M>(p)) return -1;
  if (!io) return fail("backward: null io");
  if (p->B == 0) return 0;  // empty batch: nothing to launch (empty arrays may be NULL)
  if (!io->C || !io->X || !io->U || !io->dc || (M::NTH > 0 && !io->theta))
    return fail("backward: required pointer is NULL");
  if ((io->dtheta || io->dLdJ) && !io->c) return fail("backward: c is required for dtheta / dL/dJ");
  BwdArgs a;
  memset(&a, 0, sizeof a);
  a.B = p->B; a.T = p->T; a.theta_stride = p->theta_stride; a.n_theta = p->n_theta; a.dt = p->dt;
  for (int i = 0; i < 8; i++) {
    a.u_min[i] = p->u_min[i]; a.u_max[i] = p->u_max[i];
  }
  a.theta = io->theta; a.C = io->C; a.c = io->c; a.X = io->X; a.U = io->U;
  a.dLdX = io->dLdX; a.dLdU = io->dLdU; a.dLdJ = io->dLdJ;
  a.dC = io->dC; a.dc = io->dc; a.dx0 = io->dx0; a.dtheta = io->dtheta; a.dX = io->dX; a.dU = io->dU;
  a.fail_t = io->fail_t;
  auto kern = ilqr_backward_kernel<M, G, DIAG, R>;
  if constexpr (sizeof(R) == 4) {
    if (p->T == 10) kern = ilqr_backward_kernel<M, G, DIAG, R, 10>;
  }
  using BL = BwdLayout<M, DIAG, R>;
  const BL bl = BL::make(p->T);
  a.ab = (io->dtheta != nullptr && p->n_theta > 0) || io->dLdJ != nullptr;  // co-state recursions
  if (plan<BL>(kern, p->B, p->T, G, a.gpb, a.smem_stride, nullptr, a.ab ? bl.total_ab : bl.total)) return -1;
  const int smem = a.gpb * a.smem_stride;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int blocks = (p->B + a.gpb - 1) / a.gpb;
  void* kw = nullptr;
  if constexpr (BL::kLean) {  // auxiliary gain workspace, stream-ordered
    const size_t kb = (size_t)p->B * p->T * M::NU * Dims<M, DIAG, R>::LDA * sizeof(R);
    if (cudaMallocFromPoolAsync(&kw, kb, work_pool(), s) != cudaSuccess)
      return fail("backward: gain workspace allocation of %zu bytes failed", kb);
    a.Kg = kw;
  }
  kern<<<blocks, a.gpb * G, smem, s>>>(a);
  if (kw) cudaFreeAsync(kw, s);
  g_launches.fetch_add(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail("backward launch failed: %s", cudaGetErrorString(e));
  return 0;
}

// batched dynamics: one thread per point
template <class M, class R>
__global__ void dynamics_kernel(int N, int stride, double dt, const R* theta, const R* x, const R* u,
                                R* xn, R* A, R* Bm) {
  constexpr int NX = M::NX, NU = M::NU;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const R* th = theta + (size_t)stride * i;
  R xr[NX], ur[NU];
#pragma unroll
  for (int a = 0; a < NX; a++) xr[a] = x[(size_t)i * NX + a];
#pragma unroll
  for (int a = 0; a < NU; a++) ur[a] = u[(size_t)i * NU + a];
  R* Ai = A ? A + (size_t)i * NX * NX : nullptr;
  R* Bi = Bm ? Bm + (size_t)i * NX * NU : nullptr;
  if constexpr (M::kLinearParams) {
    if (xn) {
#pragma unroll
      for (int a = 0; a < NX; a++) {
        R acc = R(0);
#pragma unroll
        for (int b = 0; b < NX; b++) acc += th[a * NX + b] * xr[b];
#pragma unroll
        for (int b = 0; b < NU; b++) acc += th[NX * NX + a * NU + b] * ur[b];
        xn[(size_t)i * NX + a] = acc;
      }
    }
    if (Ai && Bi) {
      for (int e = 0; e < NX * NX; e++) Ai[e] = th[e];
      for (int e = 0; e < NX * NU; e++) Bi[e] = th[NX * NX + e];
    }
  } else {
    R thr[M::NTH > 0 ? M::NTH : 1], P[M::NP];
#pragma unroll
    for (int a = 0; a < M::NTH; a++) thr[a] = th[a];
    M::template prep<R>(thr, P);
    if (xn) {
      R o[NX];
      M::template step<R>(P, (R)dt, xr, ur, o);
#pragma unroll
      for (int a = 0; a < NX; a++) xn[(size_t)i * NX + a] = o[a];
    }
    if (Ai && Bi) {
      M::template jac_const<R>(P, (R)dt, Ai, NX, Bi, NU, 0, 1);
      M::template jac_vary<R>(P, (R)dt, xr, ur, Ai, NX, Bi, NU);
    }
  }
}

template <class M, class R>
int dyn_impl(const DiffMPCProblem* p, int N, const void* theta, const void* x, const void* u, void* xn,
             void* A, void* Bm, cudaStream_t s) {
  if (check_theta<M>(p)) return -1;
  if (N <= 0) return 0;
  if (!x || !u || (M::NTH > 0 && !theta)) return fail("dynamics: required pointer is NULL");
  const int threads = 128, blocks = (N + threads - 1) / threads;
  dynamics_kernel<M, R><<<blocks, threads, 0, s>>>(N, p->theta_stride, p->dt, (const R*)theta,
                                                   (const R*)x, (const R*)u, (R*)xn, (R*)A, (R*)Bm);
  g_launches.fetch_add(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail("dynamics launch failed: %s", cudaGetErrorString(e));
  return 0;
}

enum class Op { Fwd, Bwd, Dyn };

struct Call {
  Op op;
  const DiffMPCProblem* p;
  const DiffMPCForwardIO* fio;
  const DiffMPCBackwardIO* bio;
  int N;
  const void *theta, *x, *u;
  void *xn, *A, *Bm;
  cudaStream_t s;
};

template <class M, class R, int G>
int run_g(const Call& c) {
  const bool diag = c.p->cost_layout == DIFFMPC_COST_DIAG;
  switch (c.op) {
    case Op::Fwd:
      return diag ? fwd_impl<M, G, true, R>(c.p, c.fio, c.s) : fwd_impl<M, G, false, R>(c.p, c.fio, c.s);
    case Op::Bwd:
      return diag ? bwd_impl<M, G, true, R>(c.p, c.bio, c.s) : bwd_impl<M, G, false, R>(c.p, c.bio, c.s);
    default:
      return dyn_impl<M, R>(c.p, c.N, c.theta, c.x, c.u, c.xn, c.A, c.Bm, c.s);
  }
}

// Lanes per problem: the default per model, or DIFFMPC_GROUP={4,8,16} (tuning / A-B).
template <class M>
int pick_group() {
  const int env = group_env();
  if (env == 4) return 4;
  if (env == 8 && M::NX > 4) return 8;
  if (env == 16 && M::NX > 8) return 16;
  return default_group(M::NX);
}

template <class M, class R>
int run(const Call& c) {
  const int g = pick_group<M>();
  if constexpr (M::NX > 8) {
    if (g == 16) return run_g<M, R, 16>(c);
  }
  if constexpr (M::NX > 4) {
    if (g == 8) return run_g<M, R, 8>(c);
  }
  return run_g<M, R, 4>(c);
}

}  // namespace dmpc

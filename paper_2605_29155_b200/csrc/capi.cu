// capi.cu — the extern "C" boundary of libdiffmpc.so (declared in include/diffmpc.h).
//
// Validates the problem (the reference's ConfigError cases, ilqr.py:43-54), picks the
// compiled (model, n_x, n_u) instantiation, sizes the launch (problems per block
// from the shared-memory footprint) and enqueues exactly ONE kernel per call on the
// caller's stream. Nothing here synchronises the stream.
#include <mutex>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/diffmpc.h"
#include "launch.cuh"

using namespace dmpc;

// The kernels are instantiated in the per-model units inst_<model>_<dtype>.cu.
namespace dmpc {
#define DMPC_CASE(KIND, NX_, NU_, MODEL)                 \
  extern template int run<MODEL, float>(const Call&);   \
  extern template int run<MODEL, double>(const Call&);
#include "instances.inc"
#undef DMPC_CASE
}  // namespace dmpc

namespace dmpc {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

int fail(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
int fail(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return -1;
}

int group_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DIFFMPC_GROUP");
    v = e ? atoi(e) : 0;
  }
  return v;
}

int num_sms() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 1;
  }
  return v;
}

cudaMemPool_t work_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[128] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
      cudaGetLastError();
      cudaDeviceGetDefaultMemPool(&pools[dev], dev);
    } else {
      uint64_t keep = UINT64_MAX;  // never trim: a per-call workspace is reused at no cost
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
      // no hidden cross-stream waits: a call on one stream must not be made to wait for the
      // release point of a workspace freed on another (pipelined streams would serialise);
      // the pool grows by one workspace per concurrently active stream instead
      int no = 0;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolReuseAllowInternalDependencies, &no);
    }
  }
  return pools[dev];
}

int max_smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0)
      v = 48 * 1024;
  }
  return v;
}

}  // namespace dmpc

namespace {

int check_problem(const DiffMPCProblem* p) {
  if (!p) return fail("null problem");
  if (p->B < 0) return fail("batch size must be >= 0, got %d", p->B);
  if (p->T < 1) return fail("horizon T must be >= 1, got %d", p->T);
  if (p->K_max < 1) return fail("K_max must be >= 1, got %d", p->K_max);
  if (p->nu < 1 || p->nu > DIFFMPC_MAX_NU) return fail("n_u=%d outside [1, %d]", p->nu, DIFFMPC_MAX_NU);
  if (p->n_alpha < 1 || p->n_alpha > DIFFMPC_MAX_ALPHA)
    return fail("n_alpha=%d outside [1, %d]", p->n_alpha, DIFFMPC_MAX_ALPHA);
  for (int i = 0; i < p->nu; i++)
    if (!(p->u_min[i] < p->u_max[i])) return fail("u_min must be elementwise below u_max");
  for (int i = 0; i < p->n_alpha; i++) {
    if (!(p->alphas[i] > 0.0 && p->alphas[i] <= 1.0))
      return fail("alphas must be a strictly decreasing sequence in (0, 1]");
    if (i > 0 && !(p->alphas[i] < p->alphas[i - 1]))
      return fail("alphas must be a strictly decreasing sequence in (0, 1]");
  }
  if (!(p->dt > 0.0)) return fail("dt must be positive");
  if (p->cost_layout != DIFFMPC_COST_DENSE && p->cost_layout != DIFFMPC_COST_DIAG)
    return fail("unknown cost layout %d", p->cost_layout);
  if (p->theta_stride != 0 && p->theta_stride != p->n_theta)
    return fail("theta_stride must be 0 or n_theta");
  if (p->kernel_select < DIFFMPC_KERNEL_AUTO || p->kernel_select > DIFFMPC_KERNEL_LATENCY)
    return fail("unknown kernel_select %d", p->kernel_select);
  return 0;
}

// (kind, nx, nu) -> instantiation. Returns 1 if handled (result in *rc).
template <class R>
bool dispatch(const Call& c, int* rc) {
  const int k = c.p->model_kind, nx = c.p->nx, nu = c.p->nu;
#define DMPC_CASE(KIND, NX_, NU_, MODEL)                      \
  if (k == KIND && nx == NX_ && nu == NU_) {                  \
    *rc = run<MODEL, R>(c);                                   \
    return true;                                              \
  }
#include "instances.inc"
#undef DMPC_CASE
  return false;
}

bool supported(int k, int nx, int nu) {
#define DMPC_CASE(KIND, NX_, NU_, MODEL) \
  if (k == KIND && nx == NX_ && nu == NU_) return true;
#include "instances.inc"
#undef DMPC_CASE
  return false;
}

template <class R>
int entry(const Call& c) {
  if (check_problem(c.p)) return -1;
  int rc = 0;
  if (!dispatch<R>(c, &rc))
    return fail("no compiled kernels for model kind %d with n_x=%d, n_u=%d", c.p->model_kind, c.p->nx, c.p->nu);
  return rc;
}

}  // namespace

extern "C" {

int diffmpc_forward_f32(const DiffMPCProblem* p, const DiffMPCForwardIO* io, void* stream) {
  Call c{Op::Fwd, p, io, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, (cudaStream_t)stream};
  return entry<float>(c);
}
int diffmpc_forward_f64(const DiffMPCProblem* p, const DiffMPCForwardIO* io, void* stream) {
  Call c{Op::Fwd, p, io, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, (cudaStream_t)stream};
  return entry<double>(c);
}
int diffmpc_backward_f32(const DiffMPCProblem* p, const DiffMPCBackwardIO* io, void* stream) {
  Call c{Op::Bwd, p, nullptr, io, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, (cudaStream_t)stream};
  return entry<float>(c);
}
int diffmpc_backward_f64(const DiffMPCProblem* p, const DiffMPCBackwardIO* io, void* stream) {
  Call c{Op::Bwd, p, nullptr, io, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, (cudaStream_t)stream};
  return entry<double>(c);
}
int diffmpc_dynamics_f32(const DiffMPCProblem* p, int32_t N, const void* theta, const void* x, const void* u,
                         void* xn, void* A, void* Bm, void* stream) {
  Call c{Op::Dyn, p, nullptr, nullptr, N, theta, x, u, xn, A, Bm, (cudaStream_t)stream};
  return entry<float>(c);
}
int diffmpc_dynamics_f64(const DiffMPCProblem* p, int32_t N, const void* theta, const void* x, const void* u,
                         void* xn, void* A, void* Bm, void* stream) {
  Call c{Op::Dyn, p, nullptr, nullptr, N, theta, x, u, xn, A, Bm, (cudaStream_t)stream};
  return entry<double>(c);
}
uint64_t diffmpc_forward_workspace_bytes(const DiffMPCProblem* p, int32_t elem_bytes) {
  if (!p || (elem_bytes != 4 && elem_bytes != 8) || p->B < 0 || p->T < 1) return 0;
  return (uint64_t)fwd_workspace_bytes(p->B, p->T, p->nx, p->nu, elem_bytes, p->cost_layout == DIFFMPC_COST_DIAG);
}
int diffmpc_supported(int32_t model_kind, int32_t nx, int32_t nu) { return supported(model_kind, nx, nu) ? 1 : 0; }
int64_t diffmpc_launch_count(void) { return g_launches.load(); }
const char* diffmpc_last_error(void) { return g_last_error.c_str(); }
int32_t diffmpc_abi_version(void) { return DIFFMPC_ABI_VERSION; }

}  // extern "C"

// raceenv.cu — the batched gate-racing environment step as ONE kernel.
//
// One thread per environment: drone dynamics (the same model code the iLQR kernels use,
// models.cuh, float64), gate-plane crossing, pass / miss / out-of-bounds / timeout
// termination, the shaped reward and the next observation, for all N environments in a
// single launch (the eager tensor version issued ~40 kernels per step). Per environment
// it follows /root/reference/pkg/src/fusedmpc/raceenv.py:174-228 (env_step) and :120-140
// (observation) term for term, in the same evaluation order, so the planar environment is
// bit-level comparable with the reference's golden vectors. The 3-D variant (13-state
// quadrotor, kind 3) is the same logic with circular gate openings (a crossing counts when
// the crossing point lies within width/2 of the gate centre in the gate plane) and the
// 19-value observation documented in raceenv.py; the reference has no 3-D environment.
//
// Environments that are already done are not advanced (the reference raises on them);
// their reward is 0 and their observation is re-emitted.
#include <cuda_runtime.h>

#include <atomic>

#include "../../include/diffmpc.h"
#include "models.cuh"

namespace dmpc {
int fail(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
}

namespace {

using namespace dmpc;

struct Layout2 {  // planar: x = [px, py, theta, vx, vy, omega]
  static constexpr int D = 2, P0 = 0, V0 = 3, OBS = 11;
};
struct Layout3 {  // 13-state: x = [p(3), q(4), v(3), w(3)]
  static constexpr int D = 3, P0 = 0, V0 = 7, OBS = 19;
};

template <class M, class L>
__global__ void race_step_kernel(const DiffMPCTrack trk, int N, double dt, const double* __restrict__ theta,
                                 double* __restrict__ x, int64_t* __restrict__ gate, int64_t* __restrict__ laps,
                                 double* __restrict__ t, uint8_t* __restrict__ done, int64_t* __restrict__ reason,
                                 const double* __restrict__ u, double* __restrict__ reward,
                                 double* __restrict__ obs) {
  constexpr int NX = M::NX, NU = M::NU, D = L::D;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double xs[NX];
#pragma unroll
  for (int a = 0; a < NX; a++) xs[a] = x[(size_t)i * NX + a];
  int64_t gi = gate[i];
  if (!done[i]) {
    double th[M::NTH], P[M::NP], us[NU], xn[NX];
#pragma unroll
    for (int a = 0; a < M::NTH; a++) th[a] = theta[a];
    M::template prep<double>(th, P);
#pragma unroll
    for (int a = 0; a < NU; a++) us[a] = u[(size_t)i * NU + a];
    M::template step<double>(P, dt, xs, us, xn);
    const double t_new = t[i] + dt;
    const double* c = trk.center[gi];
    const double* n = trk.normal[gi];
    double rew = -trk.time_penalty * dt;
    int64_t nxt = gi, lp = laps[i];
    int why = DIFFMPC_RACE_NONE;
    bool fin = true;
#pragma unroll
    for (int a = 0; a < NX; a++) fin = fin && isfinite(xn[a]);
    if (!fin) {  // raceenv.py:190-193
#pragma unroll
      for (int a = 0; a < NX; a++) xn[a] = isfinite(xn[a]) ? xn[a] : 0.0;
      why = DIFFMPC_RACE_OUT_OF_BOUNDS;
      rew -= trk.crash_penalty;
    } else {
      const double* pp = xs + L::P0;
      const double* pn = xn + L::P0;
      double dp = 0.0, dn = 0.0, sp = 0.0, sn = 0.0;
#pragma unroll
      for (int a = 0; a < D; a++) {
        dp += (pp[a] - c[a]) * (pp[a] - c[a]);
        dn += (pn[a] - c[a]) * (pn[a] - c[a]);
        sp += n[a] * (pp[a] - c[a]);
        sn += n[a] * (pn[a] - c[a]);
      }
      const double progress = trk.k_p * (sqrt(dp) - sqrt(dn));
      rew += fmin(fmax(progress, -trk.progress_cap), trk.progress_cap);
      // gate-plane crossing in the normal direction (raceenv.py:161-171)
      const bool crossed = (sp <= 0.0) && (sn > 0.0);
      double lateral = 0.0;
      if (crossed) {
        const double frac = (sn != sp) ? sp / (sp - sn) : 0.0;
        double pc[D];
#pragma unroll
        for (int a = 0; a < D; a++) pc[a] = pp[a] + frac * (pn[a] - pp[a]);
        if constexpr (D == 2) {
          lateral = fabs(-n[1] * (pc[0] - c[0]) + n[0] * (pc[1] - c[1]));
        } else {  // distance from the centre within the gate plane
          double along = 0.0;
#pragma unroll
          for (int a = 0; a < D; a++) along += n[a] * (pc[a] - c[a]);
          double r2 = 0.0;
#pragma unroll
          for (int a = 0; a < D; a++) {
            const double w = (pc[a] - c[a]) - along * n[a];
            r2 += w * w;
          }
          lateral = sqrt(r2);
        }
      }
      const double hw = trk.width[gi] / 2.0;
      bool in_b = true;
#pragma unroll
      for (int a = 0; a < D; a++) in_b = in_b && (pn[a] >= trk.lo[a]) && (pn[a] <= trk.hi[a]);
      if (crossed && lateral <= hw) {
        rew += trk.gate_bonus;
        nxt += 1;
        if (nxt == trk.n_gates) {
          lp += 1;
          nxt = 0;
          if (lp >= trk.laps) why = DIFFMPC_RACE_LAP_COMPLETE;
        }
      } else if (crossed && lateral <= trk.miss_factor * hw) {
        why = DIFFMPC_RACE_GATE_MISSED;
        rew -= trk.crash_penalty;
      } else if (!in_b) {
        why = DIFFMPC_RACE_OUT_OF_BOUNDS;
        rew -= trk.crash_penalty;
      }
      if (why == DIFFMPC_RACE_NONE && t_new >= trk.timeout) why = DIFFMPC_RACE_TIMEOUT;
    }
#pragma unroll
    for (int a = 0; a < NX; a++) {
      xs[a] = xn[a];
      x[(size_t)i * NX + a] = xn[a];
    }
    gi = nxt;
    gate[i] = nxt;
    laps[i] = lp;
    t[i] = t_new;
    reason[i] = why;
    done[i] = why != DIFFMPC_RACE_NONE;
    reward[i] = rew;
  } else {
    reward[i] = 0.0;
  }
  if (!obs) return;
  // observation of the (new) state and gate (raceenv.py:120-140; 3-D: see raceenv.py)
  const double* c1 = trk.center[gi];
  const double* n1 = trk.normal[gi];
  const double* c2 = trk.center[(gi + 1) % trk.n_gates];
  const double* p = xs + L::P0;
  double* o = obs + (size_t)i * L::OBS;
  const double ps = trk.pos_scale, vs = trk.vel_scale, ws = trk.omega_scale;
  if constexpr (D == 2) {
    o[0] = (c1[0] - p[0]) * ps;
    o[1] = (c1[1] - p[1]) * ps;
    o[2] = n1[0];
    o[3] = n1[1];
    o[4] = (c2[0] - p[0]) * ps;
    o[5] = (c2[1] - p[1]) * ps;
    o[6] = xs[3] * vs;
    o[7] = xs[4] * vs;
    o[8] = sin(xs[2]);
    o[9] = cos(xs[2]);
    o[10] = xs[5] * ws;
  } else {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      o[a] = (c1[a] - p[a]) * ps;
      o[3 + a] = n1[a];
      o[6 + a] = (c2[a] - p[a]) * ps;
      o[9 + a] = xs[L::V0 + a] * vs;
      o[16 + a] = xs[10 + a] * ws;
    }
#pragma unroll
    for (int a = 0; a < 4; a++) o[12 + a] = xs[3 + a];
  }
}

template <class M, class L>
int launch(const DiffMPCTrack* trk, int N, double dt, const double* theta, double* x, int64_t* gate, int64_t* laps,
           double* t, uint8_t* done, int64_t* reason, const double* u, double* reward, double* obs,
           cudaStream_t s) {
  const int threads = 128, blocks = (N + threads - 1) / threads;
  race_step_kernel<M, L><<<blocks, threads, 0, s>>>(*trk, N, dt, theta, x, gate, laps, t, done, reason, u, reward,
                                                    obs);
  return 0;
}

}  // namespace

namespace dmpc {
extern std::atomic<int64_t> g_launches;
}

extern "C" int diffmpc_race_step_f64(const DiffMPCTrack* trk, int32_t model_kind, int32_t N, double dt,
                                     const double* theta, double* x, int64_t* gate, int64_t* laps, double* t,
                                     uint8_t* done, int64_t* reason, const double* u, double* reward, double* obs,
                                     void* stream) {
  if (!trk) return dmpc::fail("race_step: null track");
  if (trk->n_gates < 2 || trk->n_gates > DIFFMPC_RACE_MAX_GATES)
    return dmpc::fail("race_step: n_gates=%d outside [2, %d]", trk->n_gates, DIFFMPC_RACE_MAX_GATES);
  if (N < 0) return dmpc::fail("race_step: N must be >= 0");
  if (N == 0) return 0;
  if (!theta || !x || !gate || !laps || !t || !done || !reason || !u || !reward)
    return dmpc::fail("race_step: required pointer is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if (model_kind == DIFFMPC_KIND_PLANAR_QUADROTOR && trk->dim == 2) {
    rc = launch<PlanarQuad, Layout2>(trk, N, dt, theta, x, gate, laps, t, done, reason, u, reward, obs, s);
  } else if (model_kind == DIFFMPC_KIND_QUADROTOR13 && trk->dim == 3) {
    rc = launch<Quad13, Layout3>(trk, N, dt, theta, x, gate, laps, t, done, reason, u, reward, obs, s);
  } else {
    return dmpc::fail("race_step: model kind %d with a %d-D track is not supported (planar: 2-D, "
                      "quadrotor13: 3-D)", model_kind, trk->dim);
  }
  dmpc::g_launches.fetch_add(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dmpc::fail("race_step launch failed: %s", cudaGetErrorString(e));
  return rc;
}

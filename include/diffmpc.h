/*
 * diffmpc.h — C ABI of the B200-native differentiable-MPC layer (libdiffmpc.so).
 *
 * This is the drop-in boundary for the DiffMPC hot path of arxiv/paper_2605_29155
 * (reference: /root/reference/pkg/src/fusedmpc). Every entry point takes plain
 * pointers and sizes — no torch types — so any host (Python ctypes, C++, the
 * reference's own MpcSolveLayer) can bind it. See INTEGRATION.md for bindings.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/fusedmpc):
 *   diffmpc_forward_*   <- batchexec.solve_raw (batchexec.py:156-163) driving
 *                          ilqr.run_staged_solve (ilqr.py:154-247) over the range
 *                          kernels rollout/linearize/backward/linesearch
 *                          (kernels.py:161-187, 326-512, 520-574) and the host
 *                          epilogue (ilqr.py:216-244); result semantics of
 *                          ilqr.collect_result (ilqr.py:250-268).
 *   diffmpc_backward_*  <- MpcSolveLayer.backward relinearisation (policy.py:257-272)
 *                          + batchexec.backward_batch_arrays (batchexec.py:180-186)
 *                          -> gradlayer.run_staged_backward (gradlayer.py:98-150)
 *                          over kernels.aux_backward/aux_rollout/aux_assemble
 *                          (kernels.py:582-756); plus the dynamics-parameter and
 *                          optimal-cost gradients (SURVEY.md §8(a) NEW rows).
 *   diffmpc_dynamics_*  <- kernels.step_one / jac_one (kernels.py:43-117) as used by
 *                          dynamics.step / dynamics.jacobians (dynamics.py:102-133).
 *
 * Conventions
 *   - All array pointers are DEVICE pointers (CUDA global memory), C-contiguous,
 *     batch-major exactly like the reference workspaces (ilqr.py:84-113):
 *       x0 (B,nx)  U (B,T,nu)  X (B,T+1,nx)  C (B,T,nz,nz) | diag (B,T,nz)
 *       c (B,T,nz) K (B,T,nu,nx) k (B,T,nu) ...
 *   - The _f32 entry points take float arrays, _f64 double arrays (the element type
 *     of every `void*` below). Status/flag arrays are int32 / uint8 as declared.
 *   - Stream-ordered: work is enqueued on `stream` (a cudaStream_t; NULL = legacy
 *     default stream); no host synchronisation happens inside. Reentrant per stream.
 *   - Return value: 0 = enqueued; <0 = configuration error (bad dims, unsupported
 *     model/shape, bad settings), with a message from diffmpc_last_error().
 *     Per-problem numeric failures never fail the call; they are reported through
 *     fail_t / diverged / converged exactly as the reference does (kernels.py:168-178,
 *     383-385, 468-471; ilqr.py:200, 235-236).
 */
#ifndef DIFFMPC_H
#define DIFFMPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DIFFMPC_ABI_VERSION 2

/* Model kinds. 0-2 follow dynamics.py:25-27 / kernels.py:24-26; 3 is the 13-state /
 * 4-rotor quadrotor that BASELINE.json names (no reference; defined in DESIGN.md). */
#define DIFFMPC_KIND_DOUBLE_INTEGRATOR 0
#define DIFFMPC_KIND_PLANAR_QUADROTOR  1
#define DIFFMPC_KIND_LINEAR            2
#define DIFFMPC_KIND_QUADROTOR13       3

/* Cost layouts: dense C_t (B,T,nz,nz) as batchexec.solve_raw takes it, or the AC-MPC
 * diagonal parameterisation (B,T,nz) that MpcSolver.solve_diag expands (policy.py:214-222). */
#define DIFFMPC_COST_DENSE 0
#define DIFFMPC_COST_DIAG  1

#define DIFFMPC_KERNEL_AUTO       0
#define DIFFMPC_KERNEL_THROUGHPUT 1
#define DIFFMPC_KERNEL_LATENCY    2

#define DIFFMPC_MAX_NU     8
#define DIFFMPC_MAX_ALPHA  8

/* Problem description (host struct, passed by pointer). Mirrors SolveSettings
 * (ilqr.py:30-60) + DynModel (dynamics.py:32-99). */
typedef struct DiffMPCProblem {
  int32_t B;               /* batch size (>= 0; 0 is a no-op, array pointers may be NULL) */
  int32_t T;               /* horizon (>= 1)                                           */
  int32_t nx, nu;          /* state / control dims                                     */
  int32_t model_kind;      /* DIFFMPC_KIND_*                                           */
  int32_t cost_layout;     /* DIFFMPC_COST_*                                           */
  int32_t K_max;           /* max iLQR iterations (>= 1)                               */
  int32_t n_alpha;         /* number of line-search step sizes (1..8)                  */
  int32_t boxqp_max_iter;  /* projected-Newton iterations per stage QP (ilqr.py:40)    */
  int32_t n_theta;         /* number of model parameters in theta                      */
  int32_t theta_stride;    /* 0: theta shared by the batch; n_theta: per problem        */
  int32_t kernel_select;   /* forward mapping: 0 auto (block-per-problem latency kernel for
                              B <= 2 x #SMs, persistent throughput kernel above), 1 always
                              throughput, 2 always latency. Both solve the same algorithm;
                              pin one when results must be bit-identical across batch sizes
                              (e.g. PPO rollout vs minibatch re-solve, trainer.py:9-12)   */
  double dt;               /* model timestep                                           */
  double conv_tol;         /* relative cost-decrease tolerance (ilqr.py:39)            */
  double boxqp_tol;        /* projected-gradient tolerance (ilqr.py:41)                */
  double u_min[DIFFMPC_MAX_NU];   /* per-dimension bounds, already broadcast (ilqr.py:56-60) */
  double u_max[DIFFMPC_MAX_NU];
  double alphas[DIFFMPC_MAX_ALPHA]; /* strictly decreasing in (0,1] (ilqr.py:52-54)     */
} DiffMPCProblem;

/* Forward solve I/O. Inputs const; any output pointer may be NULL (not written),
 * except X, U, J which are required. */
typedef struct DiffMPCForwardIO {
  const void* theta;       /* model params: (n_theta) or (B,n_theta); linear kind: [A row-major, B row-major] */
  const void* C;           /* (B,T,nz,nz) dense or (B,T,nz) diag                       */
  const void* c;           /* (B,T,nz)                                                 */
  const void* x0;          /* (B,nx)                                                   */
  const void* U_warm;      /* (B,T,nu); clipped to the bounds on entry (ilqr.py:165)   */
  void* X;                 /* out (B,T+1,nx) final nominal trajectory                  */
  void* U;                 /* out (B,T,nu)                                             */
  void* J;                 /* out (B) final cost (inf if the initial rollout diverged) */
  void* K;                 /* out (B,T,nu,nx) last computed feedback gains             */
  void* k;                 /* out (B,T,nu) last computed feedforward terms             */
  int32_t* iters;          /* out (B) iterations counted as in ilqr.py:217             */
  uint8_t* converged;      /* out (B) converged and not failed (ilqr.py:263)           */
  uint8_t* diverged;       /* out (B) rollout or all-candidates divergence (ilqr.py:200,235) */
  int32_t* fail_t;         /* out (B) -1 ok, else failing stage                        */
  uint8_t* clamped;        /* out (B,T,nu) (U<=u_min)|(U>=u_max) (ilqr.py:255)         */
  void* alpha_hist;        /* out (B,K_max) accepted alpha per iteration, 0 = no step  */
  void* J_hist;            /* out (B,K_max+1) cost after rollout and after each iteration (ilqr.py:202,244) */
  void* workspace;         /* device scratch of >= diffmpc_forward_workspace_bytes() bytes, 256-byte
                              aligned, or NULL: then the call allocates it stream-ordered
                              (cudaMallocAsync / cudaFreeAsync on `stream`)                */
  uint64_t workspace_bytes;
} DiffMPCForwardIO;

/* Implicit-differentiation backward I/O (one auxiliary LQR at the solution).
 * Seeds are dL/dX (B,T+1,nx), dL/dU (B,T,nu) and dL/dJ (B); each may be NULL (= 0).
 * Outputs may be NULL except dc. dC follows cost_layout (dense (B,T,nz,nz) or its
 * diagonal (B,T,nz), exactly what MpcSolveLayer.backward extracts, policy.py:274-276). */
typedef struct DiffMPCBackwardIO {
  const void* theta;
  const void* C;           /* same layout as the forward                                */
  const void* c;           /* (B,T,nz) — needed only for the dtheta / dL/dJ terms      */
  const void* X;           /* (B,T+1,nx) solution                                      */
  const void* U;           /* (B,T,nu)                                                 */
  const void* dLdX;        /* (B,T+1,nx) or NULL                                       */
  const void* dLdU;        /* (B,T,nu) or NULL                                         */
  const void* dLdJ;        /* (B) or NULL                                              */
  void* dC;                /* out, dense or diag                                       */
  void* dc;                /* out (B,T,nz)                                             */
  void* dx0;               /* out (B,nx)                                               */
  void* dtheta;            /* out (B,n_theta) per-problem parameter gradients, or NULL */
  void* dX;                /* out (B,T+1,nx) differential trajectory, or NULL          */
  void* dU;                /* out (B,T,nu), or NULL                                    */
  int32_t* fail_t;         /* out (B) -1 ok, else stage whose reduced Hessian was singular */
} DiffMPCBackwardIO;

/* Forward iLQR solve. One kernel launch per call (rollout + every iteration fused). */
int diffmpc_forward_f32(const DiffMPCProblem* p, const DiffMPCForwardIO* io, void* stream);
int diffmpc_forward_f64(const DiffMPCProblem* p, const DiffMPCForwardIO* io, void* stream);

/* Implicit backward. One kernel launch per call (relinearise + aux Riccati + diff
 * rollout + assembly + adjoint parameter gradients fused). */
int diffmpc_backward_f32(const DiffMPCProblem* p, const DiffMPCBackwardIO* io, void* stream);
int diffmpc_backward_f64(const DiffMPCProblem* p, const DiffMPCBackwardIO* io, void* stream);

/* Batched dynamics: xn = f(x,u), A = df/dx, Bm = df/du for N points. Any output may be NULL. */
int diffmpc_dynamics_f32(const DiffMPCProblem* p, int32_t N, const void* theta, const void* x,
                         const void* u, void* xn, void* A, void* Bm, void* stream);
int diffmpc_dynamics_f64(const DiffMPCProblem* p, int32_t N, const void* theta, const void* x,
                         const void* u, void* xn, void* A, void* Bm, void* stream);

/* ---------------------------------------------------------------------------------------
 * Batched gate-racing environment step (the AC-MPC training environment, SURVEY.md §8(f)
 * row 3). Replaces, per environment, raceenv.env_step + raceenv.observation
 * (/root/reference/pkg/src/fusedmpc/raceenv.py:120-140, 174-228) for N environments in ONE
 * kernel launch; planar quadrotor on a 2-D track (dim 2, the reference's environment) or the
 * 13-state quadrotor on a 3-D track (dim 3: circular gate openings, 19-value observation).
 * ------------------------------------------------------------------------------------- */
#define DIFFMPC_RACE_MAX_GATES 32
#define DIFFMPC_RACE_NONE           0
#define DIFFMPC_RACE_LAP_COMPLETE   1
#define DIFFMPC_RACE_GATE_MISSED    2
#define DIFFMPC_RACE_OUT_OF_BOUNDS  3
#define DIFFMPC_RACE_TIMEOUT        4

typedef struct DiffMPCTrack {
  int32_t n_gates, laps, dim;                 /* dim 2 (planar) or 3                     */
  int32_t pad_;
  double center[DIFFMPC_RACE_MAX_GATES][3];   /* gate centres (first `dim` entries)       */
  double normal[DIFFMPC_RACE_MAX_GATES][3];   /* unit normals (passing direction)         */
  double width[DIFFMPC_RACE_MAX_GATES];       /* opening width (3-D: diameter)            */
  double lo[3], hi[3];                        /* in-bounds box of the position            */
  /* RewardConfig (raceenv.py:88-99) and the observation scales (raceenv.py:30-32)        */
  double k_p, gate_bonus, crash_penalty, time_penalty, progress_cap, timeout, miss_factor;
  double pos_scale, vel_scale, omega_scale;
} DiffMPCTrack;

/* Advances every environment that is not done by one control period with controls u (N,nu)
 * (already clamped by the caller): x (N,nx), gate / laps / reason (N) int64, t (N), done (N)
 * uint8 are updated in place; reward (N) is written (0 for environments already done);
 * obs (N, 11 | 19) receives the next observation (NULL: skipped). Device pointers, float64. */
int diffmpc_race_step_f64(const DiffMPCTrack* track, int32_t model_kind, int32_t N, double dt,
                          const double* theta, double* x, int64_t* gate, int64_t* laps, double* t,
                          uint8_t* done, int64_t* reason, const double* u, double* reward, double* obs,
                          void* stream);

/* Bytes of device workspace one forward call needs (elem_bytes 4 for _f32, 8 for _f64):
 * a work counter for the persistent grid plus the L2-resident feedback gains. This is the
 * counterpart of the reference's preallocated Workspace gains arrays (ilqr.py:84-113). */
uint64_t diffmpc_forward_workspace_bytes(const DiffMPCProblem* p, int32_t elem_bytes);

/* 1 if (model_kind, nx, nu) has compiled kernels, else 0. */
int diffmpc_supported(int32_t model_kind, int32_t nx, int32_t nu);
/* Total kernel launches issued by this library since load (dispatch counter,
 * the analogue of batchexec.PoolDispatcher.count, batchexec.py:102-112). */
int64_t diffmpc_launch_count(void);
/* Message for the last configuration error on this thread. */
const char* diffmpc_last_error(void);
int32_t diffmpc_abi_version(void);
/* Measurement utility: FP32 FFMA throughput probe, blocks x 256 threads x iters x 128 FMAs
 * (the roofline denominator for the FP32 CUDA-core kernels). */
int diffmpc_probe_ffma(int blocks, int iters, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DIFFMPC_H */

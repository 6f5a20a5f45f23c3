// riccati.cuh — shared-memory layout helpers and the lane-parallel Riccati building
// blocks used by both the forward (iLQR) and backward (auxiliary LQR) kernels.
//
// Mapping: lane a < n_x of a problem's G-lane group owns ROW a of every n_x x n_x
// quantity (V_xx, Q_xx, MA) and COLUMN a of every n_u x n_x quantity (Q_ux, K).
// Operands every lane needs in full (A_t rows, MA rows, B_t rows, the K/Qux/QuuK
// columns) live in shared memory with rows padded to 16 bytes, so each row is
// fetched with 128-bit broadcast loads (LDS.128): the row-lane products issue one
// vector load per 4 (f32) FMAs instead of one scalar load per FMA.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace dmpc {

template <class R>
struct VecW {
  static constexpr int N = 16 / (int)sizeof(R);
};

__host__ __device__ constexpr int rup(int v, int a) { return (v + a - 1) / a * a; }

// Load the first N entries of a 16-byte aligned, padded smem row into registers.
template <int N, class R>
DMPC_DEV void lds_row(const R* __restrict__ p, R (&v)[N]) {
  if constexpr (sizeof(R) == 4) {
#pragma unroll
    for (int q = 0; q < (N + 3) / 4; q++) {
      const float4 t = reinterpret_cast<const float4*>(p)[q];
      const float tt[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int i = 0; i < 4; i++)
        if (q * 4 + i < N) v[q * 4 + i] = tt[i];
    }
  } else {
#pragma unroll
    for (int q = 0; q < (N + 1) / 2; q++) {
      const double2 t = reinterpret_cast<const double2*>(p)[q];
      const double tt[2] = {t.x, t.y};
#pragma unroll
      for (int i = 0; i < 2; i++)
        if (q * 2 + i < N) v[q * 2 + i] = tt[i];
    }
  }
}

// Store a row to a 16-byte aligned, padded shared row with vector stores (pads get 0).
template <int N, class R>
DMPC_DEV void sts_row(R* __restrict__ p, const R (&v)[N]) {
  if constexpr (sizeof(R) == 4) {
#pragma unroll
    for (int q = 0; q < (N + 3) / 4; q++) {
      float4 t;
      t.x = v[4 * q];
      t.y = 4 * q + 1 < N ? v[4 * q + 1] : 0.f;
      t.z = 4 * q + 2 < N ? v[4 * q + 2] : 0.f;
      t.w = 4 * q + 3 < N ? v[4 * q + 3] : 0.f;
      reinterpret_cast<float4*>(p)[q] = t;
    }
  } else {
#pragma unroll
    for (int q = 0; q < (N + 1) / 2; q++) {
      double2 t;
      t.x = v[2 * q];
      t.y = 2 * q + 1 < N ? v[2 * q + 1] : 0.0;
      reinterpret_cast<double2*>(p)[q] = t;
    }
  }
}

template <int N>
DMPC_DEV void lds_row_d(const double* __restrict__ p, double (&v)[N]) {
#pragma unroll
  for (int q = 0; q < (N + 1) / 2; q++) {
    const double2 t = reinterpret_cast<const double2*>(p)[q];
    v[2 * q] = t.x;
    if (2 * q + 1 < N) v[2 * q + 1] = t.y;
  }
}

// Padded leading dimensions (elements of R) for one model / precision.
template <class M, bool DIAG, class R>
struct Dims {
  static constexpr int NX = M::NX, NU = M::NU, NZ = NX + NU;
  static constexpr int VN = VecW<R>::N;
  static constexpr int LDA = rup(NX, VN);  // rows of A, Vx
  // rows of MA: each lane writes (and reads back with vector loads) its own row, so an
  // even number of 16-byte chunks per row (64 B at 13 f32) would put lanes a and a+2 on
  // the same banks; an odd count (80 B) spreads the 8 lanes of a 128-bit phase over all
  // 32 banks and leaves the scalar column stores 2-way instead of 8-way
  static constexpr int LDM = (LDA / VN) % 2 == 0 ? LDA + VN : LDA;
  static constexpr int LDB = rup(NU, VN);  // rows of B, NB, K^T, Qux^T, (QuuK)^T, Quu
  static constexpr int ZLD = rup(NZ, VN);  // z, c, rows of staged dense C
  static constexpr int NCSP = DIAG ? ZLD : NZ * ZLD;  // staged C_t (padded rows)
  static constexpr int NBUF = DIAG ? 2 : 1;            // staging buffers (dense: 1 to save smem)
  static constexpr int NCS = DIAG ? NZ : NZ * NZ;     // C_t in global memory
  static constexpr int REC = NCSP + ZLD;               // stage record [C_t padded | c_t padded]
  static constexpr int XLD = rup(NX, 2);   // rows of the double trajectories
  static constexpr int ULD = rup(NU, 2);
};

// Riccati scratch offsets (bytes), 16-byte aligned arrays.
template <class M, bool DIAG, class R>
struct RicLayout {
  using D = Dims<M, DIAG, R>;
  int oAs, oBs, oMA, oNB, oKT, oQuu, oqu, oVx, ozs, oR, end;
  // ab = false: no shared copy of A_t / B_t (a kernel that takes every Jacobian entry from
  // registers; As / Bs then alias the next array and must not be touched)
  __host__ __device__ static constexpr RicLayout make(int o, bool ab = true) {
    RicLayout L{};
    const int s = (int)sizeof(R);
    auto take = [&](int n) { int r = o; o = rup(o + n * s, 16); return r; };
    L.oAs = take(ab ? D::NX * D::LDM : 0);
    L.oBs = take(ab ? D::NX * D::LDB : 0);
    L.oMA = take(D::NX * D::LDM);
    L.oNB = take(D::NX * D::LDB);
    L.oKT = take(D::NX * D::LDB);
    L.oQuu = take(D::NU * D::LDB);
    L.oqu = take(D::LDB);
    L.oVx = take(D::LDA);
    L.ozs = take(D::ZLD);
    L.oR = take(D::NBUF * D::REC);  // NBUF contiguous stage records
    L.end = o;
    return L;
  }
};

template <class M, bool DIAG, class R>
struct Ric {
  using D = Dims<M, DIAG, R>;
  // QuxT (the Q_ux columns, full value update only) aliases NB, which is dead once the
  // Q_uu entries are formed.
  R *As, *Bs, *MA, *NB, *KT, *QuxT, *Quu, *qu, *Vx, *zs, *Rb;
  DMPC_DEV R* Cb(int b) const { return Rb + b * D::REC; }
  DMPC_DEV R* cb(int b) const { return Rb + b * D::REC + D::NCSP; }
  DMPC_DEV void bind(unsigned char* base, const RicLayout<M, DIAG, R>& L) {
    As = (R*)(base + L.oAs); Bs = (R*)(base + L.oBs); MA = (R*)(base + L.oMA);
    NB = (R*)(base + L.oNB); KT = (R*)(base + L.oKT); QuxT = NB;
    Quu = (R*)(base + L.oQuu); qu = (R*)(base + L.oqu);
    Vx = (R*)(base + L.oVx); zs = (R*)(base + L.ozs); Rb = (R*)(base + L.oR);
  }
};

// cp.async C_t (and c_t) into staging buffer `buf`, remapping rows to the padded stride.
template <class M, bool DIAG, class R, int G>
DMPC_DEV void stage_cost_t(const Ric<M, DIAG, R>& S, const R* Cg, const R* cg, int t, int buf, int lane) {
  using D = Dims<M, DIAG, R>;
  const R* src = Cg + (size_t)t * D::NCS;
  R* dst = S.Cb(buf);
  if constexpr (DIAG) {
    for (int e = lane; e < D::NZ; e += G) cp_async_elem_nh(dst + e, src + e);
  } else {
    // lane c copies column c of every row (compile-time row offsets, no index arithmetic);
    // the columns beyond the group width are spread over the lanes by row
    constexpr int NZ = D::NZ, ZLD = D::ZLD, GC = G < NZ ? G : NZ;
    if (lane < GC) {
#pragma unroll
      for (int r = 0; r < NZ; r++) cp_async_elem_nh(dst + r * ZLD + lane, src + r * NZ + lane);
    }
#pragma unroll
    for (int c = GC; c < NZ; c++)
#pragma unroll
      for (int r0 = 0; r0 < NZ; r0 += G)
        if (r0 + lane < NZ) cp_async_elem_nh(dst + (r0 + lane) * ZLD + c, src + (r0 + lane) * NZ + c);
  }
  if (cg) {
    const R* s2 = cg + (size_t)t * D::NZ;
    R* d2 = S.cb(buf);
    for (int e = lane; e < D::NZ; e += G) cp_async_elem_nh(d2 + e, s2 + e);
  }
}

// Alignment-preserving block copy of C_t (dense): the NZ x NZ block is copied as it lies in
// global memory (unpadded rows, pitch NZ) to Cb(buf) + off, off = the block's element offset
// within a 16-byte chunk, so every aligned 16-byte chunk of the source lands on an aligned
// chunk here: ~NZ*NZ/VN 16-byte copies instead of NZ*NZ element copies; the <= 2(VN-1) head /
// tail elements go one by one. Used by the single pass of the backward, whose consumers read
// the unpadded rows (ric_Qxx_Qux / ric_Quu_entry with CLD = NZ).
template <class R>
DMPC_DEV int blk_off(const R* p) {
  return (int)(((uintptr_t)p / sizeof(R)) & (uintptr_t)(16 / sizeof(R) - 1));
}
template <class M, bool DIAG, class R, int G>
DMPC_DEV void stage_cost_blk(const Ric<M, DIAG, R>& S, const R* Cg, int t, int buf, int lane) {
  using D = Dims<M, DIAG, R>;
  static_assert(!DIAG, "dense cost blocks only");
  constexpr int N = D::NCS, VN = 16 / (int)sizeof(R);
  static_assert(N + VN - 1 <= D::NCSP, "staging buffer holds the shifted block");
  const R* src = Cg + (size_t)t * N;
  const int off = blk_off(src);
  const int h = (VN - off) & (VN - 1);  // head elements before the first aligned chunk
  const int nv = (N - h) / VN;          // aligned chunks
  R* dst = S.Cb(buf) + off;
  // (no L2 cache hint: the hinted forms compiled, in some instantiations, to LDGSTS with a
  // descriptor register the kernel never writes -- tools/sass_desc_check.py)
#pragma unroll
  for (int m = 0; m < (N / VN + G - 1) / G; m++) {
    const int k = lane + m * G;
    if (k < nv) cp_async_16cg(dst + h + VN * k, src + h + VN * k);
  }
  if (lane < h) cp_async_elem_nh(dst + lane, src + lane);
  const int e = h + VN * nv + lane;
  if (lane < VN && e < N) cp_async_elem_nh(dst + e, src + e);
}

// Software pipeline over the per-stage cost tensors: `acquire(t)` makes C_t resident
// (issuing the prefetch of the next stage first when double-buffered); `release(t)`
// is called once every lane is done with C_t and, when single-buffered, issues the
// prefetch of the next stage into the same buffer. `step` is the traversal
// direction (-1 backward sweeps, +1 forward rollouts). With `Kg` set, the stage's
// feedback gains K_t (NU padded rows, written by this group's Riccati sweep into the
// L2-resident gain workspace) ride along as 16-byte cp.async.cg copies into `Kb`.
template <class M, bool DIAG, class R, int G, int NB = Dims<M, DIAG, R>::NBUF, bool BLK = false>
struct CostPipe {
  using D = Dims<M, DIAG, R>;
  // NB stage buffers: the caller provides NB contiguous records at S->Rb (NB >= NB)
  static constexpr int KCH = D::NU * D::LDA * (int)sizeof(R) / 16;  // 16-byte chunks of K_t
  const Ric<M, DIAG, R>* S;
  const R* Cg;
  const R* cg;
  int T, lane, step;
  const R* Kg = nullptr;  // gain workspace of this problem, [t][NU][LDA]
  R* Kb = nullptr;        // NBUF smem buffers of NU rows of LDM
  const R* Pk = nullptr;  // packed stage records [C_t padded rows | c_t padded] (REC elements)
  static constexpr int REC = D::REC;
  static constexpr int NCH = REC * (int)sizeof(R) / 16;  // 16-byte chunks per record
  DMPC_DEV int buf(int t) const { return NB == 2 ? (t & 1) : 0; }
  DMPC_DEV void issue(int t) {
    if (Pk) {  // contiguous record -> contiguous buffer: fully unrolled 16-byte copies
      const char* src = (const char*)(Pk + (size_t)t * REC) + 16 * lane;
      char* dst = (char*)S->Cb(buf(t)) + 16 * lane;
#pragma unroll
      for (int k = 0; k < (NCH + G - 1) / G; k++)
        if (k * G + lane < NCH) cp_async_16cg(dst + 16 * G * k, src + 16 * G * k);
    } else if constexpr (BLK) {
      stage_cost_blk<M, DIAG, R, G>(*S, Cg, t, buf(t), lane);
    } else {
      stage_cost_t<M, DIAG, R, G>(*S, Cg, cg, t, buf(t), lane);
    }
    if (Kg) {  // rows of LDA in the workspace -> rows of LDM here (the line search reads
               // four different K rows per 8-lane phase: 64-byte rows would collide)
      constexpr int CPR = D::LDA * (int)sizeof(R) / 16;  // 16-byte chunks per row
      const char* src = (const char*)(Kg + (size_t)t * D::NU * D::LDA);
      char* dst = (char*)(Kb + buf(t) * D::NU * D::LDM);
#pragma unroll
      for (int k = 0; k < (KCH + G - 1) / G; k++) {
        const int c = k * G + lane;
        if (c < KCH) cp_async_16cg(dst + (c / CPR) * D::LDM * (int)sizeof(R) + 16 * (c % CPR), src + 16 * c);
      }
    }
    cp_async_commit();
  }
  DMPC_DEV void start(int t0) { issue(t0); }
  DMPC_DEV void acquire(int t) {
    const int tn = t + step;
    if (NB == 2 && tn >= 0 && tn < T) {
      issue(tn);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      cp_async_wait_all();
    }
  }
  DMPC_DEV void release(int t) {
    const int tn = t + step;
    if (NB == 1 && tn >= 0 && tn < T) issue(tn);
  }
  // write the resident (padded) C_t / c_t out as packed record t (16-byte stores); later
  // sweeps stage it back with plain 16-byte copies
  DMPC_DEV void pack_out(R* dst, int t) const {
    const uint4* sr = (const uint4*)S->Cb(buf(t)) + lane;
    uint4* d = (uint4*)(dst + (size_t)t * REC) + lane;
#pragma unroll
    for (int k = 0; k < (NCH + G - 1) / G; k++)
      if (k * G + lane < NCH) d[G * k] = sr[G * k];
  }
  // BLK: unpadded rows (pitch NZ) starting at the staged block's alignment offset
  DMPC_DEV const R* C(int t) const {
    if constexpr (BLK) return S->Cb(buf(t)) + blk_off(Cg + (size_t)t * D::NCS);
    else return S->Cb(buf(t));
  }
  DMPC_DEV const R* c(int t) const { return S->cb(buf(t)); }
  DMPC_DEV const R* K(int t) const { return Kb + buf(t) * D::NU * D::LDM; }  // rows of LDM
};

// ---------------------------------------------------------------------------
// Row-lane building blocks. A lane owns the RPL rows a_k = lane + k*G (k < RPL) of
// every n_x x n_x quantity and the matching columns of the n_u x n_x ones; rows
// a_k >= n_x are padding (computed on zeros, never stored). Every shared-memory row
// fetched below is reused for all RPL rows of the lane.
// ---------------------------------------------------------------------------
template <int G, int RPL>
DMPC_DEV int row_of(int lane, int k) { return lane + k * G; }

// Entry classes of A_t: structural zero, the constant 1 (diagonal of I + dt df/dx), exactly
// dt (kinematic couplings), or state-dependent (read from the shared-memory copy). A row
// with no state-dependent entry is never loaded.
template <class M>
__host__ __device__ constexpr bool a_sd(int r, int c) {
  return M::a_nz(r, c) && !M::a_one(r, c) && !M::a_dt(r, c);
}
template <class M>
__host__ __device__ constexpr bool a_row_sd(int r) {
  bool any = false;
  for (int c = 0; c < M::NX; c++) any = any || a_sd<M>(r, c);
  return any;
}

template <class M>
__host__ __device__ constexpr bool b_row_nz(int r) {
  bool any = false;
  for (int c = 0; c < M::NU; c++) any = any || M::b_nz(r, c);
  return any;
}

// Row providers of A_t / B_t for the products: the shared-memory copy (any model), or
// register-resident rows formed from a model's per-stage JacRegs (no shared-memory loads).
template <class M, bool DIAG, class R>
struct SmemRows {
  const Ric<M, DIAG, R>& S;
  DMPC_DEV void get(int r, R (&a)[M::NX], R (&b)[M::NU]) const {
    using D = Dims<M, DIAG, R>;
    if (a_row_sd<M>(r)) lds_row<M::NX>(S.As + r * D::LDM, a);
    if (b_row_nz<M>(r)) lds_row<M::NU>(S.Bs + r * D::LDB, b);
  }
  DMPC_DEV R b(int r, int i) const { return S.Bs[r * Dims<M, DIAG, R>::LDB + i]; }  // B[r][i]
};
template <class M, class R>
struct RegRows {
  typename M::template JacRegs<R> J;
  DMPC_DEV void get(int r, R (&a)[M::NX], R (&b)[M::NU]) const { M::template jac_row<R>(J, r, a, b); }
  DMPC_DEV R b(int r, int i) const { return M::template jac_b<R>(J, r, i); }  // B[r][i], runtime column
};
// Write the state-dependent entries of A_t (and the rows of B_t) held in a RegRows to the
// shared-memory copy (the consumers that need columns of A / B read that copy); the values
// are the ones jac_vary would store.
template <class M, class R, class J>
DMPC_DEV void jac_store_rows(const J& rows, R* A, int lda, R* B, int ldb) {
#pragma unroll
  for (int r = 0; r < M::NX; r++) {
    R a[M::NX], b[M::NU];
    rows.get(r, a, b);
#pragma unroll
    for (int c = 0; c < M::NX; c++)
      if (M::a_nz(r, c) && !M::a_one(r, c) && !M::a_dt(r, c)) A[r * lda + c] = a[c];
    if (M::template b_varies<0>(r)) {
#pragma unroll
      for (int c = 0; c < M::NU; c++) B[r * ldb + c] = b[c];
    }
  }
}

template <class M, class = void>
struct has_jac_regs : std::false_type {};
template <class M>
struct has_jac_regs<M, std::void_t<typename M::template JacRegs<float>>> : std::true_type {};

template <class M, bool DIAG, class R, class Z>
DMPC_DEV auto make_rows(const Ric<M, DIAG, R>& S, const R* P, R dt, const Z& z) {
  if constexpr (has_jac_regs<M>::value) {
    RegRows<M, R> rr;
    M::template jac_regs<R>(P, dt, z, rr.J);
    return rr;
  } else {
    return SmemRows<M, DIAG, R>{S};
  }
}

// MA = V_xx A, NB = V_xx B  (kernels.py:411-421 / 629-639). Terms on structural zeros of
// A_t / B_t (M::a_nz / M::b_nz, compile-time) are skipped; the row of A is the same for
// every lane, so the skipping is uniform (no divergence).
template <class M, bool DIAG, class R, int G, int RPL, class Rows>
DMPC_DEV void ric_MA_NB(const Ric<M, DIAG, R>& S, int lane, const R (&vxx)[RPL][M::NX], R dt, const Rows& rows) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX, NU = M::NU;
  R ma[RPL][NX], nb[RPL][NU];
#pragma unroll
  for (int k = 0; k < RPL; k++) {
#pragma unroll
    for (int b = 0; b < NX; b++) ma[k][b] = R(0);
#pragma unroll
    for (int b = 0; b < NU; b++) nb[k][b] = R(0);
  }
#pragma unroll
  for (int r = 0; r < NX; r++) {
    R arow[NX], brow[NU];
    rows.get(r, arow, brow);
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const R v = vxx[k][r];
#pragma unroll
      for (int b = 0; b < NX; b++) {
        if (M::a_one(r, b)) ma[k][b] += v;
        else if (M::a_dt(r, b)) ma[k][b] += v * dt;
        else if (M::a_nz(r, b)) ma[k][b] += v * arow[b];
      }
#pragma unroll
      for (int b = 0; b < NU; b++)
        if (M::b_nz(r, b)) nb[k][b] += v * brow[b];
    }
  }
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    const int a = row_of<G, RPL>(lane, k);
    if (a < NX) {
      sts_row<NX>(S.MA + a * D::LDM, ma[k]);
      sts_row<NU>(S.NB + a * D::LDB, nb[k]);
    }
  }
}

// Q_xx row a = C_xx[a,:] + (A' V_xx A)[a,:]  (kernels.py:422-427) and Q_ux column a =
// C_ux[:,a] + sum_r B[r,:] MA[r,a] (kernels.py:428-433). A' V_xx A is evaluated as
// MA' A (V_xx is exactly symmetric), i.e. row a = sum_r MA[r,a] A[r,:]: the lane-uniform
// operand is again a row of A, so its structural zeros are skipped without divergence.
// CLD: row pitch of the staged C_t (padded ZLD, or NZ for the backward's unpadded block)
template <class M, bool DIAG, class R, int G, int RPL, int CLD = Dims<M, DIAG, R>::ZLD, class Rows>
DMPC_DEV void ric_Qxx_Qux(const Ric<M, DIAG, R>& S, const R* Cs, int lane, R (&qxx)[RPL][M::NX],
                          R (&quxc)[RPL][M::NU], R dt, const Rows& rows) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX, NU = M::NU;
  int ac[RPL];  // clamped row index (padding rows alias the last row; never stored)
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    const int a = row_of<G, RPL>(lane, k);
    ac[k] = a < NX ? a : NX - 1;
    if constexpr (DIAG) {
      const R caa = Cs[ac[k]];
#pragma unroll
      for (int bb = 0; bb < NX; bb++) qxx[k][bb] = (bb == ac[k]) ? caa : R(0);
#pragma unroll
      for (int i = 0; i < NU; i++) quxc[k][i] = R(0);
    } else {
      if constexpr (CLD == D::ZLD) {
        lds_row<NX>(Cs + ac[k] * D::ZLD, qxx[k]);
      } else {  // unaligned row: scalar loads
#pragma unroll
        for (int bb = 0; bb < NX; bb++) qxx[k][bb] = Cs[ac[k] * CLD + bb];
      }
#pragma unroll
      for (int i = 0; i < NU; i++) quxc[k][i] = Cs[(NX + i) * CLD + ac[k]];
    }
  }
#pragma unroll
  for (int r = 0; r < NX; r++) {
    R arow[NX], brow[NU];
    rows.get(r, arow, brow);
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const R mra = S.MA[r * D::LDM + ac[k]];
#pragma unroll
      for (int bb = 0; bb < NX; bb++) {
        if (M::a_one(r, bb)) qxx[k][bb] += mra;
        else if (M::a_dt(r, bb)) qxx[k][bb] += mra * dt;
        else if (M::a_nz(r, bb)) qxx[k][bb] += mra * arow[bb];
      }
#pragma unroll
      for (int i = 0; i < NU; i++)
        if (M::b_nz(r, i)) quxc[k][i] += brow[i] * mra;
    }
  }
}

// Q_uu entry (i,j) = C_uu[i,j] + sum_r B[r,i] NB[r,j]  (kernels.py:434-439)
template <class M, bool DIAG, class R, int CLD = Dims<M, DIAG, R>::ZLD, class Rows>
DMPC_DEV R ric_Quu_entry(const Ric<M, DIAG, R>& S, const R* Cs, int i, int j, const Rows& rows) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX;
  R s;
  if constexpr (DIAG) {
    s = (i == j) ? Cs[NX + i] : R(0);
  } else {
    s = Cs[(NX + i) * CLD + NX + j];
  }
#pragma unroll
  for (int r = 0; r < NX; r++)
    if (b_row_nz<M>(r)) s += rows.b(r, i) * S.NB[r * D::LDB + j];
  return s;
}

// Publish column a of K (and, for the full value update, of Qux).
template <class M, bool DIAG, class R>
DMPC_DEV void ric_publish_cols(const Ric<M, DIAG, R>& S, int a, const R (&kcol)[M::NU], const R (&quxc)[M::NU],
                               bool lean) {
  using D = Dims<M, DIAG, R>;
  constexpr int NU = M::NU;
  sts_row<NU>(S.KT + a * D::LDB, kcol);  // one vector store per lane: no bank conflicts
  if (lean) return;
  sts_row<NU>(S.QuxT + a * D::LDB, quxc);
}

// newVxx rows -> N (aliases MA) (kernels.py:499-507):
//   full:  N[a,b] = Qxx[a,b] + sum_r (K_ra (Quu K)_rb + K_ra Qux_rb) + Qux_ra K_rb
//   lean:  N[a,b] = Qxx[a,b] + sum_r Qux_ra K_rb
// The lean form is exact whenever K = -Quu_ff^-1 Qux_f on the free rows and zero on the
// clamped ones with the SAME Quu the update uses (lambda = 0 in the primal sweep; always in
// the auxiliary sweep, whose Quu is the frozen one it factorises): then
// K'Quu K = -K'Qux and the first two terms cancel. The full form (lambda > 0, rare)
// recomputes the column (Quu K)[:,b] from the published K column.
template <class M, bool DIAG, class R, int G, int RPL>
DMPC_DEV void ric_Vxx_rows(const Ric<M, DIAG, R>& S, int lane, const R (&qxx)[RPL][M::NX],
                           const R (&kcol)[RPL][M::NU], const R (&quxc)[RPL][M::NU],
                           const R (&quu)[M::NU][M::NU], bool lean) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX, NU = M::NU;
  // each lane's row is assembled in registers and stored with vector stores (a column of
  // scalar stores, one per lane-owned row, is bank-conflicted)
  R vrow[RPL][NX];
  if (lean) {
#pragma unroll
    for (int bb = 0; bb < NX; bb++) {
      R kk[NU];
      lds_row<NU>(S.KT + bb * D::LDB, kk);
#pragma unroll
      for (int k = 0; k < RPL; k++) {
        R s0 = qxx[k][bb], s1 = R(0);
#pragma unroll
        for (int r = 0; r < NU; r += 2) {
          s0 += quxc[k][r] * kk[r];
          if (r + 1 < NU) s1 += quxc[k][r + 1] * kk[r + 1];
        }
        vrow[k][bb] = s0 + s1;
      }
    }
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const int a = row_of<G, RPL>(lane, k);
      if (a < NX) sts_row<NX>(S.MA + a * D::LDM, vrow[k]);
    }
    return;
  }
#pragma unroll
  for (int bb = 0; bb < NX; bb++) {
    R kk[NU], qx[NU], kq[NU];
    lds_row<NU>(S.QuxT + bb * D::LDB, qx);
    lds_row<NU>(S.KT + bb * D::LDB, kk);
#pragma unroll
    for (int r = 0; r < NU; r++) {
      R t = R(0);
#pragma unroll
      for (int q = 0; q < NU; q++) t += quu[r][q] * kk[q];
      kq[r] = t;
    }
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      R s = qxx[k][bb];
#pragma unroll
      for (int r = 0; r < NU; r++) s += (kcol[k][r] * kq[r] + kcol[k][r] * qx[r]) + quxc[k][r] * kk[r];
      vrow[k][bb] = s;
    }
  }
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    const int a = row_of<G, RPL>(lane, k);
    if (a < NX) sts_row<NX>(S.MA + a * D::LDM, vrow[k]);
  }
}

// Lean value update straight into the lane's V_xx rows, without the symmetrisation pass:
//   V_xx[a,:] = Qxx[a,:] + sum_r Qux_ra K_r:
// for a symmetric cost block C_xx the update is symmetric in exact arithmetic (C_xx and
// V_xx symmetric => Q_xx = C_xx + A'V_xx A symmetric, and Q_xx - Q_ux' Quu^-1 Q_ux too), so
// the reference's V <- (V + V')/2 (kernels.py:510-512) only averages round-off; skipping
// it saves the row store, the column re-read and a group barrier per stage. Callers use it
// only when every C_t of the problem is symmetric and the lean form applies.
template <class M, bool DIAG, class R, int G, int RPL>
DMPC_DEV void ric_Vxx_lean_regs(const Ric<M, DIAG, R>& S, int lane, const R (&qxx)[RPL][M::NX],
                                const R (&quxc)[RPL][M::NU], R (&vxx)[RPL][M::NX]) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX, NU = M::NU;
#pragma unroll
  for (int bb = 0; bb < NX; bb++) {
    R kk[NU];
    lds_row<NU>(S.KT + bb * D::LDB, kk);
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      R s0 = qxx[k][bb], s1 = R(0);
#pragma unroll
      for (int r = 0; r < NU; r += 2) {
        s0 += quxc[k][r] * kk[r];
        if (r + 1 < NU) s1 += quxc[k][r + 1] * kk[r + 1];
      }
      vxx[k][bb] = s0 + s1;  // padding lanes (row >= NX) hold a finite copy of row NX-1; never stored
    }
  }
}

// V_xx rows = (N[a,:] + N[:,a]) / 2  (kernels.py:510-512); padding rows stay zero.
template <class M, bool DIAG, class R, int G, int RPL>
DMPC_DEV void ric_symmetrize(const Ric<M, DIAG, R>& S, int lane, R (&vxx)[RPL][M::NX]) {
  using D = Dims<M, DIAG, R>;
  constexpr int NX = M::NX;
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    const int a = row_of<G, RPL>(lane, k);
    if (a < NX) {
      R row[NX];
      lds_row<NX>(S.MA + a * D::LDM, row);
#pragma unroll
      for (int bb = 0; bb < NX; bb++) vxx[k][bb] = R(0.5) * (row[bb] + S.MA[bb * D::LDM + a]);
    } else {
#pragma unroll
      for (int bb = 0; bb < NX; bb++) vxx[k][bb] = R(0);
    }
  }
}

}  // namespace dmpc

// gs_cheb.cu -- the hot path: fused Chebyshev heat-filter steps with the Sinkhorn and
// barycenter updates folded into the last step's epilogue.
//
// Reference path:
//   HeatFilter::apply (proj/src/heat.cpp:116-131) over SparseSymMatrix::multiply
//   (proj/src/sparse.cpp:85-99), called twice per sweep by sinkhorn_many
//   (proj/src/transport.cpp:144-239) and sinkhorn_barycenter (proj/src/barycenter.cpp:45-99).
//
// Device layout ("grouped row-major"): a block of B vertex signals is stored as G = B/GW column
// groups, each an n x GW row-major array (GW = 8 doubles = 64 B per row for B >= 8). A warp
// gathers whole 64-byte neighbour rows with 128-bit loads (4 lanes x double2 per row, 8 rows per
// warp); one CTA = 64 rows x one group. Groups are independent, so a launch can cover all
// groups (matrix tile reused through L2 by the 8 group-CTAs of a row tile) or a subset.
//
// One Chebyshev step k >= 2 (heat.cpp:124-130), per row i, per column:
//     y   = sum_p vals[p] * T_{k-1}[cols[p]]        (fma chain from +0, CSR order)
//     T_k = 2 * (y - T_{k-1}[i]) - T_{k-2}[i]        (T_k overwrites T_{k-2} in place)
//     acc = fma(b_k, T_k, acc)
// Step 1: T_1 = y - T_0, acc = fma(b_1, T_1, (b_0/2) * T_0).  The last step (k = K) does not
// store T_K; its epilogue consumes acc (= p_K(L_s) x) in registers:
//     SK_PSI : psi -> colmin; W = N / max(psi, 1e-300); next T_0 = a * W; colmax|T_0|
//     SK_PHI : phi -> colmin; err += |V * phi - M|; V' = M / max(phi, 1e-300); T_0 = a * V'
//     BARY_PSI: psi -> colmin and stored for the log-domain geometric mean.
// Column reductions: min/max are order-free (atomics on order-preserving keys); the L1 error is
// a sum and goes through fixed-order per-CTA partials + a fixed-order finalise (deterministic).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "gs_internal.cuh"

namespace {

constexpr int kThreads = 256;
#ifndef GS_ROWS_PER_CTA
#define GS_ROWS_PER_CTA 4
#endif
constexpr int kRowsPerCta = GS_ROWS_PER_CTA;  // row blocks per CTA (L1 reuse across a block)
#ifndef GS_EARLY_LOADS
#define GS_EARLY_LOADS 0
#endif
constexpr bool kEarlyLoads = GS_EARLY_LOADS != 0;
#ifndef GS_GATHER_BATCH
#define GS_GATHER_BATCH 4
#endif
constexpr int kGatherBatch = GS_GATHER_BATCH;  // neighbour rows in flight per lane
#ifndef GS_PREFETCH
#define GS_PREFETCH 1
#endif
#ifndef GS_PREFETCH_STAGES
#define GS_PREFETCH_STAGES 2
#endif
constexpr bool kPrefetch = GS_PREFETCH != 0;
constexpr int kPrefetchStages = GS_PREFETCH_STAGES;
#ifndef GS_PREFETCH_IDX
#define GS_PREFETCH_IDX 0
#endif
constexpr bool kPrefetchIdx = GS_PREFETCH_IDX != 0;  // (col, val) prefetch: opt-in, not faster
constexpr int kTileRows = 32;
#ifndef GS_SMQUEUE
#define GS_SMQUEUE 0
#endif
constexpr bool kSmQueue = GS_SMQUEUE != 0;  // rows per staged block (gs_tiles.cu plan granularity)
#ifndef GS_TILE_PERSIST
#define GS_TILE_PERSIST 1
#endif
constexpr bool kTilePersist = GS_TILE_PERSIST != 0;
#ifndef GS_TILE_SMEM_BUDGET
#define GS_TILE_SMEM_BUDGET (100 * 1024)
#endif

enum StepMode { MODE_NONE = 0, MODE_SK_PSI = 1, MODE_SK_PHI = 2, MODE_BARY_PSI = 3 };

template <int GW>
struct Lay {
  static constexpr int VEC = GW >= 2 ? 2 : 1;
  static constexpr int LPR = GW / VEC;       // lanes per row
  static constexpr int RPW = 32 / LPR;       // rows per warp
  static constexpr int ROWS = (kThreads / 32) * RPW;  // rows per CTA
};

// order-preserving uint64 keys for doubles (atomic min/max of signed values)
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunkey(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}
constexpr unsigned long long KEY_POS_INF = 0xFFF0000000000000ull;  // dkey(+inf)
constexpr unsigned long long KEY_ZERO = 0x8000000000000000ull;     // dkey(+0.0)

template <int VEC>
__device__ __forceinline__ void ld_vec(const double* p, double (&v)[VEC]) {
  if constexpr (VEC == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = t.x;
    v[1] = t.y;
  } else {
    v[0] = __ldg(p);
  }
}
template <int VEC>
__device__ __forceinline__ void ld_vec_rw(const double* p, double (&v)[VEC]) {
  if constexpr (VEC == 2) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    v[0] = t.x;
    v[1] = t.y;
  } else {
    v[0] = *p;
  }
}
template <int VEC>
__device__ __forceinline__ void st_vec(double* p, const double (&v)[VEC]) {
  if constexpr (VEC == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

struct ColState {
  // per column (Bpad entries each)
  int* active;                 // nullable
  int* gactive;                // active columns per group (nullable)
  unsigned long long* cmin;    // min of the apply output
  unsigned long long* cmax;    // max |next T_0|
  double* thr;                 // positivity threshold of the current apply
  double* errcol;              // L1 marginal error
  double* part_err;            // [tiles][Bpad]
};

struct StepArgs {
  const int* __restrict__ offs;
  const int* __restrict__ cols;
  const double* __restrict__ vals;
  int n, tiles, g0, Gl, Bpad;
  const double* Tprev;  // T_{k-1}
  double* Tout;         // T_{k-2} in, T_k out (or next T_0 / SpMM output)
  double* acc;
  double bk, b0h;
  int k;                // 0 = plain SpMM into Tout
  const gs_status* status;
  ColState cs;
  // epilogue operands (grouped layout unless noted)
  const double* a;      // n
  const double* M;      // PSI: N (targets); PHI: M (sources / members)
  const double* Vcur;   // PHI: V of this sweep
  double* Wout;         // PSI: W; PHI: V of the next sweep
  int* counters;        // per-SM work queues (k_cheb_smq), nullable
  // staged-neighbour path (k_cheb_tile)
  const unsigned short* slot;
  const int* bfirst;
  const int* bcount;
  const int* rstart;
  const int* rlen;
  const int* lbase;
};

// One row of one Chebyshev step for the calling lane group; epilogue partials accumulate in
// mn/mx/er. Own-row streaming loads (T_{k-1}[i], T_{k-2}[i], acc[i], epilogue operands) are issued
// before the neighbour gathers so HBM reads overlap the gather latency.
template <int GW, int MODE, bool SMEM = false>
__device__ __forceinline__ void cheb_row(const StepArgs& A, int g, int row, int sub, int q,
                                         double (&mn)[Lay<GW>::VEC], double (&mx)[Lay<GW>::VEC],
                                         double (&er)[Lay<GW>::VEC],
                                         const double* pre = nullptr, int pre_stride = 0,
                                         const double* sx = nullptr,
                                         const int* pre_c = nullptr, const double* pre_v = nullptr,
                                         int pre_pb = 0, int pre_pe = 0) {
  using L = Lay<GW>;
  constexpr int VEC = L::VEC, LPR = L::LPR;
  const bool valid = row < A.n;
  const size_t gbase = (size_t)g * A.n * GW + q * VEC;
  const size_t idx = gbase + (size_t)(valid ? row : 0) * GW;
  const double* __restrict__ Tp = A.Tprev + gbase;
  // ---- own-row loads (before the gathers when GS_EARLY_LOADS) ------------------------------
  double tp[VEC], t2[VEC], a0[VEC], op1[VEC], op2[VEC];
  double ai = 0.0;
  auto own_loads = [&]() {
    if (valid && A.k != 0) {
      if (pre) {  // prefetched by cp.async into shared memory (k_cheb_step pipeline)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          tp[e] = pre[e];
          t2[e] = pre[pre_stride + e];
          a0[e] = pre[2 * pre_stride + e];
        }
      } else {
        ld_vec<VEC>(A.Tprev + idx, tp);
        if (A.k >= 2) {
          ld_vec_rw<VEC>(A.Tout + idx, t2);
          ld_vec_rw<VEC>(A.acc + idx, a0);
        }
      }
      if constexpr (MODE == MODE_SK_PSI || MODE == MODE_SK_PHI) {
        ld_vec<VEC>(A.M + idx, op1);
        ai = __ldg(A.a + row);
      }
      if constexpr (MODE == MODE_SK_PHI) ld_vec_rw<VEC>(A.Vcur + idx, op2);
    }
  };
  if constexpr (kEarlyLoads) own_loads();
  // ---- y = L_s T_{k-1} (row) ------------------------------------------------------------------
  double y[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) y[e] = 0.0;
  if constexpr (LPR == 1) {
    if (valid) {
      int p = __ldg(A.offs + row);
      const int pe = __ldg(A.offs + row + 1);
      for (; p + 4 <= pe; p += 4) {
        int cc[4];
        double vv[4];
        double xx[4][VEC];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cc[u] = __ldg(A.cols + p + u);
          vv[u] = __ldg(A.vals + p + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) ld_vec<VEC>(Tp + (size_t)cc[u] * GW, xx[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(vv[u], xx[u][e], y[e]);
      }
      for (; p < pe; ++p) {
        const int c = __ldg(A.cols + p);
        const double v = __ldg(A.vals + p);
        double x[VEC];
        ld_vec<VEC>(Tp + (size_t)c * GW, x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = fma(v, x[e], y[e]);
      }
    }
  } else {
    // the LPR lanes of a row load LPR consecutive (col, val) entries with one coalesced access
    // and broadcast them by shuffle; the fma chain still runs in CSR order.
    const unsigned mask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
    const int pb = pre_c ? pre_pb : (valid ? __ldg(A.offs + row) : 0);
    const int pe = pre_c ? pre_pe : (valid ? __ldg(A.offs + row + 1) : 0);
    constexpr int GB = kGatherBatch;
    // gather source: global T_{k-1} (L1/L2) or the block's staged window in shared memory
    auto gather = [&](int c, double (&x)[VEC]) {
      if constexpr (SMEM) {
        const double* p = sx + (size_t)c * GW + q * VEC;
        if constexpr (VEC == 2) {
          const double2 t = *reinterpret_cast<const double2*>(p);
          x[0] = t.x;
          x[1] = t.y;
        } else {
          x[0] = p[0];
        }
      } else {
        ld_vec<VEC>(Tp + (size_t)c * GW, x);
      }
    };
    for (int p0 = pb; p0 < pe; p0 += LPR) {
      int myc = 0;
      double myv = 0.0;
      if (p0 + q < pe) {
        if (pre_c && p0 == pb) {  // first chunk prefetched by cp.async (k_cheb_step pipeline)
          myc = pre_c[q];
          myv = pre_v[q];
        } else {
          myc = SMEM ? (int)__ldg(A.slot + p0 + q) : __ldg(A.cols + p0 + q);
          myv = __ldg(A.vals + p0 + q);
        }
      }
      const int cnt = min(LPR, pe - p0);
      int u = 0;
      constexpr int GBX = SMEM ? 8 : GB;
      for (; u + GBX <= cnt; u += GBX) {
        int cc[GBX];
        double vv[GBX];
        double xx[GBX][VEC];
#pragma unroll
        for (int j = 0; j < GBX; ++j) {
          cc[j] = __shfl_sync(mask, myc, u + j, LPR);
          vv[j] = __shfl_sync(mask, myv, u + j, LPR);
        }
#pragma unroll
        for (int j = 0; j < GBX; ++j) gather(cc[j], xx[j]);
#pragma unroll
        for (int j = 0; j < GBX; ++j)
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = fma(vv[j], xx[j][e], y[e]);
      }
      if constexpr (GBX > 4) {
        for (; u + 4 <= cnt; u += 4) {
          int cc[4];
          double vv[4];
          double xx[4][VEC];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            cc[j] = __shfl_sync(mask, myc, u + j, LPR);
            vv[j] = __shfl_sync(mask, myv, u + j, LPR);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) gather(cc[j], xx[j]);
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < VEC; ++e) y[e] = fma(vv[j], xx[j][e], y[e]);
        }
      }
      for (; u < cnt; ++u) {
        const int c = __shfl_sync(mask, myc, u, LPR);
        const double v = __shfl_sync(mask, myv, u, LPR);
        double x[VEC];
        gather(c, x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = fma(v, x[e], y[e]);
      }
    }
  }
  if (!valid) return;
  if (A.k == 0) {  // plain SpMM (sparse.cpp:85-99)
    st_vec<VEC>(A.Tout + idx, y);
    return;
  }
  if constexpr (!kEarlyLoads) own_loads();
  // ---- recurrence (heat.cpp:121-130) ----------------------------------------------------------
  double t[VEC], ac[VEC];
  if (A.k == 1) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      t[e] = y[e] - tp[e];
      ac[e] = fma(A.bk, t[e], A.b0h * tp[e]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      t[e] = 2.0 * (y[e] - tp[e]) - t2[e];
      ac[e] = fma(A.bk, t[e], a0[e]);
    }
  }
  if constexpr (MODE == MODE_NONE) {
    st_vec<VEC>(A.Tout + idx, t);
    st_vec<VEC>(A.acc + idx, ac);
  } else {
    // ---- fused epilogue of the last step ----------------------------------------------------
    const int* act = A.cs.active;
    const int col0 = g * GW + q * VEC;
#pragma unroll
    for (int e = 0; e < VEC; ++e) mn[e] = fmin(mn[e], ac[e]);
    if constexpr (MODE == MODE_SK_PSI) {
      double w[VEC], t0[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        w[e] = op1[e] / fmax(ac[e], GS_FLOOR);      // transport.cpp:180
        t0[e] = ai * w[e];                          // transport.cpp:172
        mx[e] = fmax(mx[e], fabs(t0[e]));
      }
      st_vec<VEC>(A.Tout + idx, t0);
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (!act || act[col0 + e]) A.Wout[idx + e] = w[e];
    } else if constexpr (MODE == MODE_SK_PHI) {
      double vn[VEC], t0[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        er[e] = er[e] + fabs(op2[e] * ac[e] - op1[e]);  // transport.cpp:184
        vn[e] = op1[e] / fmax(ac[e], GS_FLOOR);         // transport.cpp:178
        t0[e] = ai * vn[e];
        mx[e] = fmax(mx[e], fabs(t0[e]));
      }
      st_vec<VEC>(A.Tout + idx, t0);
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (!act || act[col0 + e]) A.Wout[idx + e] = vn[e];
    } else {  // MODE_BARY_PSI
      st_vec<VEC>(A.acc + idx, ac);
    }
  }
}

template <int GW, int MODE>
__device__ __forceinline__ void block_epilogue(const StepArgs& A, int g, int tile, int warp, int sub,
                                               int q, double (&mn)[Lay<GW>::VEC],
                                               double (&mx)[Lay<GW>::VEC],
                                               double (&er)[Lay<GW>::VEC]);

// A CTA owns RPC x (8 warps x RPW) consecutive rows of one column group; at each of its RPC
// iterations the 8 warps cover a contiguous block, so neighbouring gathers share L1 lines.
#ifndef GS_MIN_BLOCKS
#define GS_MIN_BLOCKS 1
#endif
template <int GW, int MODE, int RPC>
__global__ void __launch_bounds__(kThreads, GS_MIN_BLOCKS) k_cheb_step(const StepArgs A) {
  using L = Lay<GW>;
  constexpr int VEC = L::VEC, LPR = L::LPR, RPW = L::RPW;
  constexpr int BLOCK_ROWS = (kThreads / 32) * RPW;
  if (A.status && (A.status->error || A.status->done)) return;
  const int tile = blockIdx.x / A.Gl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = 0.0;
    er[e] = 0.0;
  }
  const int base = tile * (BLOCK_ROWS * RPC) + warp * RPW + sub;
  if constexpr (kPrefetch && VEC == 2) {
    // Own-row operands of the next row block (T_{k-1}[i], T_{k-2}[i], acc[i]) -- and, with one
    // warp per row, the row's first 32 (col, val) entries -- are copied to shared memory with
    // cp.async while this block's neighbour gathers run: DRAM/L2 reads stay in flight without
    // holding registers. Each lane reads back only what it copied itself.
    constexpr int STG = kPrefetchStages;
    constexpr bool IDX = LPR == 32 && kPrefetchIdx;
    __shared__ __align__(16) double s_pre[STG][3][kThreads * 2];
    __shared__ __align__(16) int s_col[IDX ? STG : 1][IDX ? kThreads : 1];
    __shared__ __align__(16) double s_val[IDX ? STG : 1][IDX ? kThreads : 1];
    const size_t gbase = (size_t)g * A.n * GW + q * VEC;
    // row offsets of this warp's RPC rows: lane j holds offs[row_j], offs[row_j + 1]
    int o_lo = 0, o_hi = 0;
    if constexpr (IDX) {
      const int rj = base + lane * BLOCK_ROWS;
      if (lane < RPC && rj < A.n) {
        o_lo = __ldg(A.offs + rj);
        o_hi = __ldg(A.offs + rj + 1);
      }
    }
    auto issue = [&](int j) {
      const int row = base + j * BLOCK_ROWS;
      if (j < RPC && row < A.n) {
        if (A.k != 0) {
          const size_t idx = gbase + (size_t)row * GW;
          double* d = &s_pre[j % STG][0][threadIdx.x * 2];
          cp_async16(d, A.Tprev + idx);
          if (A.k >= 2) {
            cp_async16(d + kThreads * 2, A.Tout + idx);
            cp_async16(d + 2 * kThreads * 2, A.acc + idx);
          }
        }
        if constexpr (IDX) {
          const int pb = __shfl_sync(0xffffffffu, o_lo, j), pe = __shfl_sync(0xffffffffu, o_hi, j);
          if (pb + q < pe) {
            cp_async4(&s_col[j % STG][threadIdx.x], A.cols + pb + q);
            cp_async8(&s_val[j % STG][threadIdx.x], A.vals + pb + q);
          }
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int j = 0; j < STG - 1; ++j) issue(j);
#pragma unroll 1
    for (int j = 0; j < RPC; ++j) {
      issue(j + STG - 1);
      cp_async_wait<STG - 1>();
      if constexpr (IDX) {
        const int pb = __shfl_sync(0xffffffffu, o_lo, j), pe = __shfl_sync(0xffffffffu, o_hi, j);
        cheb_row<GW, MODE>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er,
                           &s_pre[j % STG][0][threadIdx.x * 2], kThreads * 2, nullptr,
                           &s_col[j % STG][warp * 32], &s_val[j % STG][warp * 32], pb, pe);
      } else {
        cheb_row<GW, MODE>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er,
                           &s_pre[j % STG][0][threadIdx.x * 2], kThreads * 2);
      }
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < RPC; ++j) cheb_row<GW, MODE>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er);
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<GW, MODE>(A, g, tile, warp, sub, q, mn, mx, er);
}

template <int GW, int MODE>
__device__ __forceinline__ void block_epilogue(const StepArgs& A, int g, int tile, int warp, int sub,
                                               int q, double (&mn)[Lay<GW>::VEC],
                                               double (&mx)[Lay<GW>::VEC],
                                               double (&er)[Lay<GW>::VEC]) {
  using L = Lay<GW>;
  constexpr int VEC = L::VEC, LPR = L::LPR;
  {
    // warp: combine rows with the same column slot (lane bits >= log2(LPR))
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        mn[e] = fmin(mn[e], __shfl_xor_sync(0xffffffffu, mn[e], off));
        mx[e] = fmax(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], off));
        er[e] = er[e] + __shfl_xor_sync(0xffffffffu, er[e], off);
      }
    }
    __shared__ double s_mn[kThreads / 32][GW], s_mx[kThreads / 32][GW], s_er[kThreads / 32][GW];
    if (sub == 0) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        s_mn[warp][q * VEC + e] = mn[e];
        s_mx[warp][q * VEC + e] = mx[e];
        s_er[warp][q * VEC + e] = er[e];
      }
    }
    __syncthreads();
    if (threadIdx.x < GW) {
      const int c = threadIdx.x;
      double a_mn = s_mn[0][c], a_mx = s_mx[0][c], a_er = s_er[0][c];
#pragma unroll
      for (int w = 1; w < kThreads / 32; ++w) {
        a_mn = fmin(a_mn, s_mn[w][c]);
        a_mx = fmax(a_mx, s_mx[w][c]);
        a_er = a_er + s_er[w][c];
      }
      const int col = g * GW + c;
      atomicMin(A.cs.cmin + col, dkey(a_mn));
      if constexpr (MODE == MODE_SK_PSI || MODE == MODE_SK_PHI) atomicMax(A.cs.cmax + col, dkey(a_mx));
      if constexpr (MODE == MODE_SK_PHI) A.cs.part_err[(size_t)tile * A.Bpad + col] = a_er;
    }
  }
}

// ---- per-SM work queues: every SM drains a contiguous range of row blocks ---------------------
// A CTA reads %smid and takes the next block of that SM's range (then steals from the following
// SMs once its own range is empty, so completion never depends on CTA placement). All CTAs
// resident on an SM work on adjacent rows, so the Cuthill-McKee neighbour window they gather is
// shared in that SM's L1.
__device__ __forceinline__ unsigned smid_u32() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

template <int GW, int MODE, int RPC>
__global__ void __launch_bounds__(kThreads) k_cheb_smq(const StepArgs A, int* counters, int nsm) {
  using L = Lay<GW>;
  constexpr int VEC = L::VEC, LPR = L::LPR, RPW = L::RPW;
  constexpr int BLOCK_ROWS = (kThreads / 32) * RPW;
  if (A.status && (A.status->error || A.status->done)) return;
  __shared__ int s_item;
  const int total = A.tiles * A.Gl;  // items = (tile, group)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  const int home = (int)(smid_u32() % (unsigned)nsm);
  for (int probe = 0; probe < nsm; ++probe) {
    const int s = (home + probe) % nsm;
    const int lo = (int)((long long)total * s / nsm), hi = (int)((long long)total * (s + 1) / nsm);
    for (;;) {
      if (threadIdx.x == 0) s_item = lo + atomicAdd(counters + s, 1);
      __syncthreads();
      const int item = s_item;
      __syncthreads();
      if (item >= hi) break;
      const int tile = item / A.Gl, g = A.g0 + item % A.Gl;
      if (A.cs.gactive && A.cs.gactive[g] == 0) continue;
      double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        mn[e] = INFINITY;
        mx[e] = 0.0;
        er[e] = 0.0;
      }
      const int base = tile * (BLOCK_ROWS * RPC) + warp * RPW + sub;
#pragma unroll 1
      for (int j = 0; j < RPC; ++j) cheb_row<GW, MODE>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er);
      if constexpr (MODE != MODE_NONE) block_epilogue<GW, MODE>(A, g, tile, warp, sub, q, mn, mx, er);
    }
  }
}

// ---- staged-neighbour step: one CTA per (block of kTileRows rows, column group) -------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

template <int GW, int MODE>
__global__ void __launch_bounds__(kThreads) k_cheb_tile(const StepArgs A) {
  using L = Lay<GW>;
  constexpr int VEC = L::VEC, LPR = L::LPR, RPW = L::RPW;
  constexpr int BLOCK_ROWS = (kThreads / 32) * RPW;
  constexpr int PASSES = kTileRows / BLOCK_ROWS;
  static_assert(PASSES >= 1 && kTileRows % BLOCK_ROWS == 0, "tile rows");
  extern __shared__ __align__(128) double sx[];
  __shared__ __align__(8) unsigned long long mbar;
  if (A.status && (A.status->error || A.status->done)) return;
  const int b = blockIdx.x / A.Gl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const unsigned bar = smem_u32(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // stage every run of T_{k-1} rows this block references with one TMA bulk copy each
    const int first = A.bfirst[b], cnt = first < 0 ? 0 : A.bcount[b];
    unsigned bytes = 0;
    for (int r = 0; r < cnt; ++r) bytes += (unsigned)A.rlen[first + r] * GW * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
                 : "memory");
    const double* src0 = A.Tprev + (size_t)g * A.n * GW;
    for (int r = 0; r < cnt; ++r) {
      const int run = first + r;
      const double* src = src0 + (size_t)A.rstart[run] * GW;
      const unsigned dst = smem_u32(sx + (size_t)A.lbase[run] * GW);
      const unsigned sz = (unsigned)A.rlen[run] * GW * 8u;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
          "l"(src), "r"(sz), "r"(bar)
          : "memory");
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = 0.0;
    er[e] = 0.0;
  }
  // wait for the staged window (phase 0)
  {
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar)
          : "memory");
    }
  }
  const int base = b * kTileRows + warp * RPW + sub;
#pragma unroll 1
  for (int j = 0; j < PASSES; ++j)
    cheb_row<GW, MODE, true>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er, nullptr, 0, sx);
  if constexpr (MODE != MODE_NONE) block_epilogue<GW, MODE>(A, g, b, warp, sub, q, mn, mx, er);
}

// Persistent, double-buffered variant: each CTA walks (block, group) items with a stride of
// gridDim.x; TMA stages item i+1's neighbour window into the other buffer while item i computes.
template <int GW, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_cheb_tilep(const StepArgs A, int max_slots) {
  using L = Lay<GW>;
  constexpr int VEC = L::VEC, LPR = L::LPR, RPW = L::RPW;
  constexpr int BLOCK_ROWS = (kThreads / 32) * RPW;
  constexpr int PASSES = kTileRows / BLOCK_ROWS;
  extern __shared__ __align__(128) double sx[];
  __shared__ __align__(8) unsigned long long mbar[2];
  if (A.status && (A.status->error || A.status->done)) return;
  const int total = A.tiles * A.Gl;
  const size_t stage_elems = (size_t)max_slots * GW;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int item, int stage) {  // thread 0 only
    const int b = item / A.Gl, g = A.g0 + item % A.Gl;
    const bool live = !(A.cs.gactive && A.cs.gactive[g] == 0);
    const int first = A.bfirst[b], cnt = (first < 0 || !live) ? 0 : A.bcount[b];
    unsigned bytes = 0;
    for (int r = 0; r < cnt; ++r) bytes += (unsigned)A.rlen[first + r] * GW * 8u;
    const unsigned bar = smem_u32(&mbar[stage]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
                 : "memory");
    const double* src0 = A.Tprev + (size_t)g * A.n * GW;
    double* dst0 = sx + stage * stage_elems;
    for (int r = 0; r < cnt; ++r) {
      const int run = first + r;
      const double* src = src0 + (size_t)A.rstart[run] * GW;
      const unsigned dst = smem_u32(dst0 + (size_t)A.lbase[run] * GW);
      const unsigned sz = (unsigned)A.rlen[run] * GW * 8u;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
          "l"(src), "r"(sz), "r"(bar)
          : "memory");
    }
  };
  if (threadIdx.x == 0 && (int)blockIdx.x < total) issue(blockIdx.x, 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  unsigned phase[2] = {0u, 0u};
  int it = 0;
  for (int item = blockIdx.x; item < total; item += gridDim.x, ++it) {
    const int stage = it & 1;
    const int next = item + gridDim.x;
    if (threadIdx.x == 0 && next < total) issue(next, stage ^ 1);
    {
      const unsigned bar = smem_u32(&mbar[stage]);
      unsigned done = 0;
      while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase[stage])
            : "memory");
      }
      phase[stage] ^= 1u;
    }
    const int b = item / A.Gl, g = A.g0 + item % A.Gl;
    if (!(A.cs.gactive && A.cs.gactive[g] == 0)) {
      double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        mn[e] = INFINITY;
        mx[e] = 0.0;
        er[e] = 0.0;
      }
      const int base = b * kTileRows + warp * RPW + sub;
      const double* stg = sx + stage * stage_elems;
#pragma unroll 1
      for (int j = 0; j < PASSES; ++j)
        cheb_row<GW, MODE, true>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er, nullptr, 0, stg);
      if constexpr (MODE != MODE_NONE) block_epilogue<GW, MODE>(A, g, b, warp, sub, q, mn, mx, er);
    }
    __syncthreads();  // every warp is done with this stage before it is refilled
  }
}

// Per-column finalise after an apply (transport.cpp:30-38 / barycenter.cpp:14-21):
// positivity check of active columns against the threshold of this apply, threshold of the
// next apply from max|T_0|, deterministic L1 error, reset of the atomic keys.
struct FinArgs {
  ColState cs;
  int B, tiles, Bpad;
  int check, has_next, has_err;
  gs_status* status;
  int knp_code;
};

__global__ void __launch_bounds__(kThreads) k_finalize(const FinArgs F) {
  const int col = blockIdx.x;
  if (col >= F.B) return;
  __shared__ double sh[kThreads];
  double acc = 0.0;
  if (F.has_err) {
    for (int t = threadIdx.x; t < F.tiles; t += kThreads) acc = acc + F.cs.part_err[(size_t)t * F.Bpad + col];
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const bool act = !F.cs.active || F.cs.active[col];
  if (F.check && act && F.status->error == 0) {
    const double mn = dunkey(F.cs.cmin[col]);
    if (!(mn >= -F.cs.thr[col])) atomicCAS(&F.status->error, 0, F.knp_code);
  }
  if (F.has_next) F.cs.thr[col] = 1e-12 * dunkey(F.cs.cmax[col]);
  if (F.has_err) F.cs.errcol[col] = sh[0];
  F.cs.cmin[col] = KEY_POS_INF;
  F.cs.cmax[col] = KEY_ZERO;
}

// ---- Sinkhorn control (transport.cpp:184-226), one thread, columns in pair order ------------
struct CtlArgs {
  int* active;
  int* gactive;
  int GW;
  const double* errcol;
  int* iters;
  int* conv;
  int* stag;
  int* final_sweep;
  double* err_out;
  gs_status* status;
  int P, sweep, max_iter, no_abort;
  double tol;
};

__global__ void k_sk_control(const CtlArgs C) {
  gs_status* st = C.status;
  if (st->error) return;
  const int s = C.sweep;
  int na = 0;
  for (int c = 0; c < C.P; ++c) {
    if (!C.active[c]) continue;
    const double err = C.errcol[c];
    C.iters[c] = s;
    C.err_out[c] = err;
    const bool done = err <= C.tol;
    if (done) C.conv[c] = 1;
    if (done || s == C.max_iter) C.final_sweep[c] = s;
    if (!done) {
      C.stag[c] = err > 0.5 ? C.stag[c] + 1 : 0;
      if (!C.no_abort && !(C.stag[c] < 50)) {
        st->error = ERRC_DISCONNECTED + 1;
        st->fail_pair = c;
        st->fail_sweep = s;
        return;
      }
      ++na;
    } else {
      C.active[c] = 0;
      C.gactive[c / C.GW] -= 1;
    }
  }
  if (s == C.max_iter) {
    for (int c = 0; c < C.P; ++c) {
      if (C.active[c]) C.gactive[c / C.GW] -= 1;
      C.active[c] = 0;
    }
    na = 0;
  }
  st->n_active = na;
}

// ---- layout conversion -------------------------------------------------------------------
// column-major (width contiguous n-vectors) <-> grouped row-major (G x n x GW)
__global__ void k_pack(const double* __restrict__ src, double* __restrict__ dst, int n, int width,
                       int GW, int G, double fill, const int* __restrict__ order) {
  const int64_t total = (int64_t)G * n * GW;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % GW);
    const int64_t r = e / GW;
    const int i = (int)(r % n);
    const int g = (int)(r / n);
    const int col = g * GW + c;
    const int o = order ? order[i] : i;
    dst[e] = col < width ? (src ? src[(size_t)col * n + o] : fill) : 0.0;
  }
}

__global__ void k_unpack(const double* __restrict__ src, double* __restrict__ dst, int n,
                         int width, int GW, const double* __restrict__ alt,
                         const int* __restrict__ sel, const int* __restrict__ newpos) {
  const int64_t total = (int64_t)width * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(e / n);
    const int i0 = (int)(e % n);
    const int i = newpos ? newpos[i0] : i0;
    const int g = col / GW, c = col % GW;
    const size_t idx = ((size_t)g * n + i) * GW + c;
    const double* s = (alt && sel && (sel[col] & 1)) ? alt : src;
    dst[e] = s[idx];
  }
}

// T_0 = a * 1 for the initial phi apply (transport.cpp:171-176 with W = 1), colmax |T_0|
__global__ void k_sk_init(const double* __restrict__ a, double* __restrict__ T0, int n, int GW,
                          int G, int B, unsigned long long* cmax) {
  const int64_t total = (int64_t)G * n * GW;
  double local = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % GW);
    const int i = (int)((e / GW) % n);
    const int col = (int)((e / GW) / n) * GW + c;
    const double v = col < B ? a[i] * 1.0 : 0.0;
    T0[e] = v;
    if (col < B) local = fmax(local, fabs(v));
  }
  // all columns share max|a|; fold into every real column's key
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = local;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < B; ++c) atomicMax(cmax + c, dkey(sh[0]));
}

// ---- validation (transport.cpp:56-66, 96-102; barycenter.cpp:32-43) ----------------------------
// per column: deterministic sum, any non-finite, any negative (first-failure order is resolved on
// the host in the reference's check order).
__global__ void k_validate_cols(const double* __restrict__ X, int n, double* sums, int* nonfinite,
                                int* negative) {
  const int col = blockIdx.y;
  const double* x = X + (size_t)col * n;
  __shared__ double sh[kThreads];
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  double total = 0.0;
  // chunks processed sequentially by the CTA: lane t folds c*4096 + j*256 + t, tree per chunk,
  // chunk partials folded in order by lane 0 (deterministic).
  for (int64_t c = 0; c < nchunks; ++c) {
    double acc = 0.0;
    int bad_f = 0, bad_n = 0;
    for (int j = 0; j < DET_J; ++j) {
      const int64_t i = c * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
      if (i < n) {
        const double v = x[i];
        if (!isfinite(v)) bad_f = 1;
        if (v < 0.0) bad_n = 1;
        acc = acc + v;
      }
    }
    if (bad_f) atomicExch(nonfinite + col, 1);
    if (bad_n) atomicExch(negative + col, 1);
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) total = total + sh[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[col] = total;
}

__global__ void k_validate_weights(const double* __restrict__ a, int n, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !(a[i] > 0.0)) atomicExch(bad, 1);
}

// ---- final cost / KL (transport.cpp:137-140, 229-237) ------------------------------------
// partials over DET chunks x columns, then a fixed-order fold per column.
__global__ void k_sk_cost_partial(const double* __restrict__ a, const double* __restrict__ M,
                                  const double* __restrict__ N, const double* __restrict__ V0,
                                  const double* __restrict__ V1, const double* __restrict__ W,
                                  const int* __restrict__ final_sweep, int n, int GW,
                                  double* part /* [chunks][P][4] */, int P) {
  const int col = blockIdx.y;
  const int64_t c = blockIdx.x;
  const int g = col / GW, cc = col % GW;
  const double* V = (final_sweep[col] & 1) ? V1 : V0;
  double s[4] = {0, 0, 0, 0};
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = c * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i >= n) break;
    const size_t idx = ((size_t)g * n + i) * GW + cc;
    const double mu = M[idx], nu = N[idx], ai = a[i];
    if (mu > 0.0) {
      const double lv = log(V[idx]);
      s[0] = s[0] + ai * mu * lv;
      s[2] = s[2] + mu * lv;
    }
    if (nu > 0.0) {
      const double w = W[idx];
      s[1] = s[1] + ai * nu * log(w);
      s[3] = s[3] + nu * log(fmax(ai * w, GS_FLOOR));
    }
  }
  __shared__ double sh[4][kThreads];
#pragma unroll
  for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int st = kThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
#pragma unroll
      for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = sh[q][threadIdx.x] + sh[q][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x < 4) part[((size_t)c * P + col) * 4 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void k_sk_cost_final(const double* part, int64_t nchunks, int P, double lambda,
                                double* cost, double* kl) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= P) return;
  double s[4] = {0, 0, 0, 0};
  for (int64_t c = 0; c < nchunks; ++c)
    for (int q = 0; q < 4; ++q) s[q] = s[q] + part[((size_t)c * P + col) * 4 + q];
  cost[col] = lambda * (s[0] + s[1]);
  kl[col] = s[2] + s[3] - 1.0;
}

// ---- barycenter row kernels (barycenter.cpp:75-84) -------------------------------------------
__global__ void k_bary_lb(const double* __restrict__ psi, const double* __restrict__ alphas,
                          int n, int m, int GW, double* __restrict__ lb, const gs_status* st) {
  if (st->error || st->done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int c = 0; c < m; ++c) {
    const double v = psi[((size_t)(c / GW) * n + i) * GW + (c % GW)];
    const double ps = fmin(fmax(v, GS_FLOOR), GS_CEIL);
    acc = fma(alphas[c], log(ps), acc);
  }
  lb[i] = acc;
}

__global__ void k_max_key(const double* __restrict__ x, int n, unsigned long long* key) {
  double local = -INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    local = fmax(local, x[i]);
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = local;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(key, dkey(sh[0]));
}

// bary_i = exp(lb_i - max) with DET-chunk partial sums of the mass
__global__ void k_bary_exp(const double* __restrict__ lb, const unsigned long long* maxkey,
                           int n, double* __restrict__ bary, double* part, const gs_status* st) {
  if (st->error || st->done) return;
  const double mx = dunkey(*maxkey);
  double acc = 0.0;
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = (int64_t)blockIdx.x * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i < n) {
      const double b = exp(lb[i] - mx);
      bary[i] = b;
      acc = acc + b;
    }
  }
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// DET-chunk partial sums of an n-vector (one chunk of 4096 per CTA)
__global__ void k_chunk_sum(const double* __restrict__ x, int n, double* part) {
  double acc = 0.0;
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = (int64_t)blockIdx.x * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i < n) acc = acc + x[i];
  }
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// deterministic fold of chunk partials (lane t folds t, t+256, ... then the tree)
__global__ void k_fold(const double* part, int64_t nparts, double* out) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < nparts; q += kThreads) acc = acc + part[q];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void k_bary_mass_check(const double* mass, gs_status* st) {
  if (st->error || st->done) return;
  if (!(*mass > 0.0)) st->error = 1000 + ERRC_KERNEL_NOT_POSITIVE + 1;  // "collapsed" variant
}

// bary /= mass; W_c = bary / max(psi_c, 1e-300); T_0 = a * W_c; colmax |T_0|
__global__ void k_bary_w(double* __restrict__ bary, const double* __restrict__ mass,
                         const double* __restrict__ psi, const double* __restrict__ a, int n,
                         int m, int GW, double* __restrict__ W, double* __restrict__ T0,
                         unsigned long long* cmax, const gs_status* st) {
  if (st->error || st->done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double ms = *mass;
  if (i < n) {
    const double b = bary[i] / ms;
    bary[i] = b;
    const double ai = a[i];
    for (int c = 0; c < m; ++c) {
      const size_t idx = ((size_t)(c / GW) * n + i) * GW + (c % GW);
      const double w = b / fmax(psi[idx], GS_FLOOR);
      W[idx] = w;
      const double t0 = ai * w;
      T0[idx] = t0;
      atomicMax(cmax + c, dkey(fabs(t0)));
    }
  }
}

// err = max over (local) members; optional hook in between; then the decision.
__global__ void k_bary_errlocal(const double* errcol, int m, double* errbuf) {
  double e = 0.0;
  for (int c = 0; c < m; ++c) e = fmax(e, errcol[c]);
  *errbuf = e;
}

__global__ void k_bary_control(const double* errbuf, gs_status* st, int sweep, double tol,
                               int* iters, int* conv, double* err_out, int max_iter) {
  if (st->error || st->done) return;
  const double err = *errbuf;
  *err_out = err;
  *iters = sweep;
  if (err <= tol) {
    *conv = 1;
    st->done = 1;
  } else if (sweep == max_iter) {
    st->done = 2;
  }
}

__global__ void k_scale_div(double* x, const double* s, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] / *s;
}

__global__ void k_fill(double* x, int64_t n, double v) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    x[e] = v;
}

__global__ void k_fill_key(unsigned long long* x, int n, unsigned long long v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

__global__ void k_gather(const double* __restrict__ src, const int* __restrict__ order, int n,
                         double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[order[i]];
}

__global__ void k_scale_vals(double* v, int64_t nnz, double scale) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) v[e] = v[e] * scale;
}

inline unsigned grid_for(int64_t work, int threads = kThreads) {
  int64_t b = (work + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

// Columns per group: the next power of two >= B, at most 64 (one warp per 512-byte row).
int choose_gw(int width) {
  int g = 1;
  while (g < width && g < 64) g <<= 1;
  return g;
}

int rows_per_cta(int gw) {
  switch (gw) {
    case 64: return Lay<64>::ROWS * kRowsPerCta;
    case 32: return Lay<32>::ROWS * kRowsPerCta;
    case 16: return Lay<16>::ROWS * kRowsPerCta;
    case 8: return Lay<8>::ROWS * kRowsPerCta;
    case 4: return Lay<4>::ROWS * kRowsPerCta;
    case 2: return Lay<2>::ROWS * kRowsPerCta;
    default: return Lay<1>::ROWS * kRowsPerCta;
  }
}

template <int GW, int MODE>
void launch_smq_mode(const StepArgs& A, int* counters, cudaStream_t s) {
  constexpr int RPC = kRowsPerCta;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cheb_smq<GW, MODE, RPC>, kThreads, 0);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaMemsetAsync(counters, 0, nsm * sizeof(int), s);
  k_cheb_smq<GW, MODE, RPC><<<(unsigned)(nsm * std::max(per_sm, 1)), kThreads, 0, s>>>(A, counters, nsm);
}

template <int GW>
void launch_step_gw(const StepArgs& A, int mode, cudaStream_t s) {
  constexpr int RPC = kRowsPerCta;
  if (kSmQueue && A.counters) {
    switch (mode) {
      case MODE_NONE: launch_smq_mode<GW, MODE_NONE>(A, A.counters, s); break;
      case MODE_SK_PSI: launch_smq_mode<GW, MODE_SK_PSI>(A, A.counters, s); break;
      case MODE_SK_PHI: launch_smq_mode<GW, MODE_SK_PHI>(A, A.counters, s); break;
      default: launch_smq_mode<GW, MODE_BARY_PSI>(A, A.counters, s); break;
    }
    return;
  }
  dim3 grid((unsigned)(A.tiles * A.Gl));
  switch (mode) {
    case MODE_NONE: k_cheb_step<GW, MODE_NONE, RPC><<<grid, kThreads, 0, s>>>(A); break;
    case MODE_SK_PSI: k_cheb_step<GW, MODE_SK_PSI, RPC><<<grid, kThreads, 0, s>>>(A); break;
    case MODE_SK_PHI: k_cheb_step<GW, MODE_SK_PHI, RPC><<<grid, kThreads, 0, s>>>(A); break;
    default: k_cheb_step<GW, MODE_BARY_PSI, RPC><<<grid, kThreads, 0, s>>>(A); break;
  }
}

template <int GW, int MODE>
void launch_tile_mode(const StepArgs& A, size_t smem, cudaStream_t s) {
  if constexpr (kTilePersist) {
    static size_t configured = 0;
    const size_t sm2 = 2 * smem;
    if (sm2 > 48 * 1024 && sm2 > configured) {
      cudaFuncSetAttribute(k_cheb_tilep<GW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      configured = sm2;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cheb_tilep<GW, MODE>, kThreads, sm2);
    if (per_sm < 1) per_sm = 1;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int total = A.tiles * A.Gl;
    const int grid = std::min(total, nsm * per_sm);
    k_cheb_tilep<GW, MODE><<<(unsigned)std::max(grid, 1), kThreads, sm2, s>>>(A, (int)(smem / (GW * 8)));
  } else {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      cudaFuncSetAttribute(k_cheb_tile<GW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured = smem;
    }
    k_cheb_tile<GW, MODE><<<(unsigned)(A.tiles * A.Gl), kThreads, smem, s>>>(A);
  }
}

template <int GW>
void launch_tile_gw(const StepArgs& A, int mode, size_t smem, cudaStream_t s) {
  switch (mode) {
    case MODE_NONE: launch_tile_mode<GW, MODE_NONE>(A, smem, s); break;
    case MODE_SK_PSI: launch_tile_mode<GW, MODE_SK_PSI>(A, smem, s); break;
    case MODE_SK_PHI: launch_tile_mode<GW, MODE_SK_PHI>(A, smem, s); break;
    default: launch_tile_mode<GW, MODE_BARY_PSI>(A, smem, s); break;
  }
}

void launch_tile(gs_ctx* ctx, int gw, const StepArgs& A, int mode, size_t smem) {
  gs_launch_begin(ctx, 0);
  switch (gw) {
    case 64: launch_tile_gw<64>(A, mode, smem, ctx->stream); break;
    case 32: launch_tile_gw<32>(A, mode, smem, ctx->stream); break;
    default: launch_tile_gw<16>(A, mode, smem, ctx->stream); break;
  }
  gs_launch_end(ctx, 0);
}

void launch_step(gs_ctx* ctx, int gw, const StepArgs& A, int mode) {
  gs_launch_begin(ctx, 0);
  switch (gw) {
    case 64: launch_step_gw<64>(A, mode, ctx->stream); break;
    case 32: launch_step_gw<32>(A, mode, ctx->stream); break;
    case 16: launch_step_gw<16>(A, mode, ctx->stream); break;
    case 8: launch_step_gw<8>(A, mode, ctx->stream); break;
    case 4: launch_step_gw<4>(A, mode, ctx->stream); break;
    case 2: launch_step_gw<2>(A, mode, ctx->stream); break;
    default: launch_step_gw<1>(A, mode, ctx->stream); break;
  }
  gs_launch_end(ctx, 0);
}

// Workspace for one batched run: grouped buffers + per-column state.
struct Work {
  int n = 0, B = 0, GW = 1, G = 1, Bpad = 1, tiles = 0;
  bool tile = false;     // staged-neighbour kernel (k_cheb_tile)
  size_t tile_smem = 0;
  DevBuf<double> T[2], acc;
  DevBuf<unsigned long long> cmin, cmax;
  DevBuf<double> thr, errcol, part_err;
  DevBuf<int> active, gactive, counters;
  DevBuf<gs_status> status;
  int init(gs_ctx* ctx, int n_, int B_, bool want_err, const gs_filter* f = nullptr) {
    cudaStream_t s = ctx->stream;
    n = n_;
    B = B_;
    GW = choose_gw(B);
    const char* env = getenv("GS_TILE");
    // staged-neighbour path: experimental, opt-in with GS_TILE=1 (slower than k_cheb_step so far;
    // profiles/r01_summary.md)
    tile = f && f->tiles.max_slots > 0 && GW >= 16 && env && env[0] == '1';
    if (tile) {
      while (GW > 16 && (size_t)f->tiles.max_slots * GW * 8 > (size_t)GS_TILE_SMEM_BUDGET) GW >>= 1;
      tile_smem = (size_t)f->tiles.max_slots * GW * 8;
      if (tile_smem > (size_t)GS_TILE_SMEM_BUDGET) tile = false;
    }
    G = (B + GW - 1) / GW;
    Bpad = G * GW;
    tiles = tile ? f->tiles.nblocks : (n + rows_per_cta(GW) - 1) / rows_per_cta(GW);
    const size_t len = (size_t)Bpad * n;
    GS_CUDA(ctx, T[0].alloc(len, s));
    GS_CUDA(ctx, T[1].alloc(len, s));
    GS_CUDA(ctx, acc.alloc(len, s));
    GS_CUDA(ctx, cmin.alloc(Bpad, s));
    GS_CUDA(ctx, cmax.alloc(Bpad, s));
    GS_CUDA(ctx, thr.alloc(Bpad, s));
    GS_CUDA(ctx, errcol.alloc(Bpad, s));
    GS_CUDA(ctx, part_err.alloc(want_err ? (size_t)tiles * Bpad : 1, s));
    GS_CUDA(ctx, active.alloc(Bpad, s));
    GS_CUDA(ctx, counters.alloc(1024, s));
    GS_CUDA(ctx, gactive.alloc(G, s));
    {
      std::vector<int> ga(G);
      for (int g = 0; g < G; ++g) ga[g] = std::min(GW, B - g * GW);
      GS_CUDA(ctx, cudaMemcpyAsync(gactive.get(), ga.data(), G * sizeof(int), cudaMemcpyHostToDevice, s));
      GS_CUDA(ctx, cudaStreamSynchronize(s));
    }
    GS_CUDA(ctx, status.alloc(1, s));
    GS_CUDA(ctx, cudaMemsetAsync(status.get(), 0, sizeof(gs_status), s));
    GS_CUDA(ctx, cudaMemsetAsync(thr.get(), 0, Bpad * sizeof(double), s));
    GS_CUDA(ctx, cudaMemsetAsync(errcol.get(), 0, Bpad * sizeof(double), s));
    k_fill_key<<<grid_for(Bpad), kThreads, 0, s>>>(cmin.get(), Bpad, KEY_POS_INF);
    k_fill_key<<<grid_for(Bpad), kThreads, 0, s>>>(cmax.get(), Bpad, KEY_ZERO);
    return GS_OK;
  }
  ColState cs() {
    ColState c;
    c.active = active.get();
    c.gactive = gactive.get();
    c.cmin = cmin.get();
    c.cmax = cmax.get();
    c.thr = thr.get();
    c.errcol = errcol.get();
    c.part_err = part_err.get();
    return c;
  }
};

// Runs one full filter application on the workspace: T0 in T[a0]; K steps; the last step uses
// `mode` with the given epilogue operands. Returns the buffer index holding the next T_0.
int run_apply(gs_ctx* ctx, const gs_filter* f, Work& w, int a0, int mode, const double* a,
              const double* M, const double* Vcur, double* Wout, bool use_active,
              bool use_status) {
  const gs_graph* S = f->perm;
  const int K = f->degree;
  StepArgs A{};
  A.offs = S->offs;
  A.cols = S->cols;
  A.vals = S->vals;
  A.n = w.n;
  A.tiles = w.tiles;
  A.g0 = 0;
  A.Gl = w.G;
  A.Bpad = w.Bpad;
  A.acc = w.acc.get();
  A.b0h = f->coeffs[0] / 2.0;
  A.status = use_status ? w.status.get() : nullptr;
  A.cs = w.cs();
  if (!use_active) {
    A.cs.active = nullptr;
    A.cs.gactive = nullptr;
  }
  A.a = a;
  A.M = M;
  A.Vcur = Vcur;
  A.Wout = Wout;
  A.counters = w.counters.get();
  A.slot = f->tiles.slot;
  A.bfirst = f->tiles.bfirst;
  A.bcount = f->tiles.bcount;
  A.rstart = f->tiles.rstart;
  A.rlen = f->tiles.rlen;
  A.lbase = f->tiles.lbase;
  for (int k = 1; k <= K; ++k) {
    A.k = k;
    A.bk = f->coeffs[k];
    A.Tprev = w.T[(a0 + k - 1) & 1].get();
    A.Tout = w.T[(a0 + k) & 1].get();
    if (w.tile) launch_tile(ctx, w.GW, A, k == K ? mode : MODE_NONE, w.tile_smem);
    else launch_step(ctx, w.GW, A, k == K ? mode : MODE_NONE);
  }
  return (a0 + K) & 1;
}

void run_finalize(gs_ctx* ctx, Work& w, int check, int has_next, int has_err, int knp_code,
                  bool use_active) {
  FinArgs F{};
  F.cs = w.cs();
  if (!use_active) F.cs.active = nullptr;
  F.B = w.B;
  F.tiles = w.tiles;
  F.Bpad = w.Bpad;
  F.check = check;
  F.has_next = has_next;
  F.has_err = has_err;
  F.status = w.status.get();
  F.knp_code = knp_code;
  gs_launch_begin(ctx, 1);
  k_finalize<<<w.B, kThreads, 0, ctx->stream>>>(F);
  gs_launch_end(ctx, 1);
}

}  // namespace

// ============================================================================================
// HeatFilter (heat.cpp:72-96): scaled Laplacian copy + coefficients, both on the device.
// ============================================================================================
extern "C" int gs_filter_create(gs_ctx* ctx, const gs_graph* L, int kind, double lambda_bound,
                                double t, int degree, gs_filter** out) {
  *out = nullptr;
  if (!(t > 0.0 && std::isfinite(t))) return gs_fail(ctx, ERRC_NON_POSITIVE_TIME, "diffusion time must be > 0");
  if (degree < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "Chebyshev degree must be >= 1");
  double scale;
  if (kind == GS_LAPLACIAN_NORMALIZED) {
    scale = 1.0;
  } else {
    if (!(lambda_bound >= 0.0 && std::isfinite(lambda_bound)))
      return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "bad lambda_max_bound");
    scale = lambda_bound > 1e-300 ? 2.0 / lambda_bound : 1.0;
  }
  gs_filter* f = new gs_filter();
  f->t = t;
  f->scale = scale;
  f->t_eff = t / scale;
  f->degree = degree;
  f->kind = kind;
  f->coeffs.assign(degree + 1, 0.0);
  int rc = gs_graph_alloc(ctx, L->n, L->nnz, &f->scaled);
  if (!rc) {
    cudaStream_t s = ctx->stream;
    cudaMemcpyAsync(f->scaled->offs, L->offs, ((size_t)L->n + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(f->scaled->cols, L->cols, (size_t)L->nnz * sizeof(int), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(f->scaled->vals, L->vals, (size_t)L->nnz * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (L->nnz > 0) {
      gs_launch_begin(ctx, 1);
      k_scale_vals<<<(unsigned)((L->nnz + 255) / 256), 256, 0, s>>>(f->scaled->vals, L->nnz, scale);
      gs_launch_end(ctx, 1);
    }
    if (cudaMalloc((void**)&f->d_coeffs, (degree + 1) * sizeof(double)) != cudaSuccess)
      rc = gs_fail(ctx, ERRC_INVALID_ARGUMENT, "coefficient allocation failed");
  }
  if (!rc) rc = gs_coefficients_impl(ctx, f->t_eff, degree, f->d_coeffs, f->coeffs.data());
  if (!rc) {
    const int n = L->n;
    if (cudaMalloc((void**)&f->order, ((size_t)n + 1) * sizeof(int)) != cudaSuccess ||
        cudaMalloc((void**)&f->newpos, ((size_t)n + 1) * sizeof(int)) != cudaSuccess)
      rc = gs_fail(ctx, ERRC_INVALID_ARGUMENT, "permutation allocation failed");
  }
  if (!rc) rc = gs_bfs_order(ctx, f->scaled, f->order, f->newpos);
  if (!rc) rc = gs_permute_graph(ctx, f->scaled, f->order, f->newpos, &f->perm);
  if (!rc) {
    rc = gs_tiles_build(ctx, f->perm, kTileRows, &f->tiles);
    if (!rc && f->tiles.max_slots >= 65536) gs_tiles_release(f->tiles);  // 16-bit slots only
  }
  if (rc) {
    gs_filter_destroy(f);
    return rc;
  }
  *out = f;
  return GS_OK;
}

extern "C" void gs_filter_destroy(gs_filter* f) {
  if (!f) return;
  gs_graph_destroy(f->scaled);
  gs_graph_destroy(f->perm);
  gs_tiles_release(f->tiles);
  cudaFree(f->order);
  cudaFree(f->newpos);
  cudaFree(f->d_coeffs);
  delete f;
}

extern "C" int gs_filter_info(const gs_filter* f, int* n, double* t, double* t_eff, double* scale,
                              int* degree, int* kind) {
  if (n) *n = f->scaled->n;
  if (t) *t = f->t;
  if (t_eff) *t_eff = f->t_eff;
  if (scale) *scale = f->scale;
  if (degree) *degree = f->degree;
  if (kind) *kind = f->kind;
  return GS_OK;
}

extern "C" int gs_filter_coefficients(const gs_filter* f, double* out) {
  memcpy(out, f->coeffs.data(), f->coeffs.size() * sizeof(double));
  return GS_OK;
}

extern "C" const gs_graph* gs_filter_scaled(const gs_filter* f) { return f->scaled; }

extern "C" int gs_filter_order(gs_ctx* ctx, const gs_filter* f, int* order, int mem) {
  GS_TRY(gs_copy_out(ctx, order, f->order, (size_t)f->scaled->n * sizeof(int), mem));
  return gs_ctx_synchronize(ctx);
}

// Input staging: returns a device pointer to `count` doubles (the caller's when mem = DEVICE).
static int stage_in(gs_ctx* ctx, DevBuf<double>& buf, const double* src, size_t count, int mem,
                    const double** out) {
  if (mem == GS_MEM_DEVICE) {
    *out = src;
    return GS_OK;
  }
  GS_CUDA(ctx, buf.alloc(count, ctx->stream));
  GS_CUDA(ctx, cudaMemcpyAsync(buf.get(), src, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  *out = buf.get();
  return GS_OK;
}

static int finish_out(gs_ctx* ctx, DevBuf<double>& buf, double* dst, size_t count, int mem) {
  if (mem == GS_MEM_DEVICE) return GS_OK;
  GS_CUDA(ctx, cudaMemcpyAsync(dst, buf.get(), count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  return GS_OK;
}

// heat.cpp:116-131
extern "C" int gs_filter_apply(gs_ctx* ctx, const gs_filter* f, const double* X, double* Y,
                               int width, int mem) {
  const int n = f->scaled->n;
  if (width < 0) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "width");
  if (width == 0 || n == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  Work w;
  GS_TRY(w.init(ctx, n, width, false, f));
  DevBuf<double> xin, yout;
  const double* dX = nullptr;
  GS_TRY(stage_in(ctx, xin, X, (size_t)width * n, mem, &dX));
  double* dY = Y;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, yout.alloc((size_t)width * n, s));
    dY = yout.get();
  }
  gs_launch_begin(ctx, 1);
  k_pack<<<grid_for((int64_t)w.Bpad * n), kThreads, 0, s>>>(dX, w.T[0].get(), n, width, w.GW, w.G, 0.0, f->order);
  gs_launch_end(ctx, 1);
  run_apply(ctx, f, w, 0, MODE_NONE, nullptr, nullptr, nullptr, nullptr, false, false);
  gs_launch_begin(ctx, 1);
  k_unpack<<<grid_for((int64_t)width * n), kThreads, 0, s>>>(w.acc.get(), dY, n, width, w.GW, nullptr, nullptr, f->newpos);
  gs_launch_end(ctx, 1);
  GS_TRY(finish_out(ctx, yout, Y, (size_t)width * n, mem));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// sparse.cpp:70-99
extern "C" int gs_graph_multiply(gs_ctx* ctx, const gs_graph* g, const double* x, double* y,
                                 int width, int mem) {
  const int n = g->n;
  if (width <= 0 || n == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  Work w;
  GS_TRY(w.init(ctx, n, width, false));
  DevBuf<double> xin, yout;
  const double* dX = nullptr;
  GS_TRY(stage_in(ctx, xin, x, (size_t)width * n, mem, &dX));
  double* dY = y;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, yout.alloc((size_t)width * n, s));
    dY = yout.get();
  }
  gs_launch_begin(ctx, 1);
  k_pack<<<grid_for((int64_t)w.Bpad * n), kThreads, 0, s>>>(dX, w.T[0].get(), n, width, w.GW, w.G, 0.0, nullptr);
  gs_launch_end(ctx, 1);
  StepArgs A{};
  A.offs = g->offs;
  A.cols = g->cols;
  A.vals = g->vals;
  A.n = n;
  A.tiles = w.tiles;
  A.Gl = w.G;
  A.Bpad = w.Bpad;
  A.k = 0;
  A.Tprev = w.T[0].get();
  A.Tout = w.T[1].get();
  launch_step(ctx, w.GW, A, MODE_NONE);
  gs_launch_begin(ctx, 1);
  k_unpack<<<grid_for((int64_t)width * n), kThreads, 0, s>>>(w.T[1].get(), dY, n, width, w.GW, nullptr, nullptr, nullptr);
  gs_launch_end(ctx, 1);
  GS_TRY(finish_out(ctx, yout, y, (size_t)width * n, mem));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// ============================================================================================
// Geodesic Sinkhorn batch (transport.cpp:108-255)
// ============================================================================================
static int validate_columns(gs_ctx* ctx, const double* d, int n, int P, std::vector<double>& sums,
                            std::vector<int>& nonfinite, std::vector<int>& negative) {
  cudaStream_t s = ctx->stream;
  DevBuf<double> dsum;
  DevBuf<int> dnf, dng;
  GS_CUDA(ctx, dsum.alloc(P, s));
  GS_CUDA(ctx, dnf.alloc(P, s));
  GS_CUDA(ctx, dng.alloc(P, s));
  GS_CUDA(ctx, cudaMemsetAsync(dnf.get(), 0, P * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(dng.get(), 0, P * sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_validate_cols<<<dim3(1, P), kThreads, 0, s>>>(d, n, dsum.get(), dnf.get(), dng.get());
  gs_launch_end(ctx, 1);
  sums.resize(P);
  nonfinite.resize(P);
  negative.resize(P);
  GS_CUDA(ctx, cudaMemcpyAsync(sums.data(), dsum.get(), P * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(nonfinite.data(), dnf.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(negative.data(), dng.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// Distribution::validate (transport.cpp:96-102) for column p
static int check_distribution(gs_ctx* ctx, int n, double sum, int nonfinite, int negative) {
  if (n < 1) return gs_fail(ctx, ERRC_LENGTH_MISMATCH, "empty distribution");
  if (nonfinite) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "non-finite weights");
  if (negative) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "negative weights");
  if (!(std::fabs(sum - 1.0) <= 1e-12)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "distribution must sum to 1");
  return GS_OK;
}

static int check_weights(gs_ctx* ctx, const double* da, int n) {
  DevBuf<int> bad;
  GS_CUDA(ctx, bad.alloc(1, ctx->stream));
  GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0, sizeof(int), ctx->stream));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_validate_weights<<<(n + 255) / 256, 256, 0, ctx->stream>>>(da, n, bad.get());
    gs_launch_end(ctx, 1);
  }
  int h = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return h ? gs_fail(ctx, ERRC_INVALID_ARGUMENT, "vertex weights must be positive") : GS_OK;
}

static const char* kKnpTransport =
    "heat approximation produced negative mass; increase the degree or diffusion time";
static const char* kKnpBary =
    "heat filter produced negative mass; increase the Chebyshev degree or diffusion time";

extern "C" int gs_sinkhorn(gs_ctx* ctx, const gs_filter* f, const double* a, const double* mus,
                           const double* nus, int P, int max_iter, double tol, int flags, int mem,
                           double* out_v, double* out_w, double* out_cost, double* out_kl,
                           int* out_iters, int* out_conv, double* out_err, int* fail_pair,
                           int* fail_sweep) {
  if (fail_pair) *fail_pair = -1;
  if (fail_sweep) *fail_sweep = 0;
  const int n = f->scaled->n;
  cudaStream_t s = ctx->stream;
  if (P < 0) return gs_fail(ctx, ERRC_SIZE_MISMATCH, "pair lists differ in length");
  if (P == 0) return GS_OK;
  // ---- stage + validate (check_transport_inputs, transport.cpp:56-66) -------------------------
  DevBuf<double> bmu, bnu, ba;
  const double *dmu, *dnu, *da;
  GS_TRY(stage_in(ctx, bmu, mus, (size_t)P * n, mem, &dmu));
  GS_TRY(stage_in(ctx, bnu, nus, (size_t)P * n, mem, &dnu));
  GS_TRY(stage_in(ctx, ba, a, (size_t)n, mem, &da));
  const double* da_user = da;
  {
    std::vector<double> smu, snu;
    std::vector<int> fmu, gmu, fnu, gnu;
    GS_TRY(validate_columns(ctx, dmu, n, P, smu, fmu, gmu));
    GS_TRY(validate_columns(ctx, dnu, n, P, snu, fnu, gnu));
    int bad_a = -1;
    for (int p = 0; p < P; ++p) {
      GS_TRY(check_distribution(ctx, n, smu[p], fmu[p], gmu[p]));
      GS_TRY(check_distribution(ctx, n, snu[p], fnu[p], gnu[p]));
      if (bad_a < 0) {
        const int rc = check_weights(ctx, da_user, n);
        if (rc) return rc;
        bad_a = 0;
      }
      if (!(tol > 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "tolerance must be positive");
      if (max_iter < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "max_iter must be >= 1");
    }
  }
  // vertex weights in the filter's locality order
  DevBuf<double> aperm;
  GS_CUDA(ctx, aperm.alloc(n, s));
  gs_launch_begin(ctx, 1);
  k_gather<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(da_user, f->order, n, aperm.get());
  gs_launch_end(ctx, 1);
  da = aperm.get();
  // ---- workspace -----------------------------------------------------------------------------
  Work w;
  GS_TRY(w.init(ctx, n, P, true, f));
  const size_t len = (size_t)w.Bpad * n;
  DevBuf<double> M, N, V[2], W;
  GS_CUDA(ctx, M.alloc(len, s));
  GS_CUDA(ctx, N.alloc(len, s));
  GS_CUDA(ctx, V[0].alloc(len, s));
  GS_CUDA(ctx, V[1].alloc(len, s));
  GS_CUDA(ctx, W.alloc(len, s));
  DevBuf<int> iters, conv, stag, final_sweep;
  DevBuf<double> errv;
  GS_CUDA(ctx, iters.alloc(w.Bpad, s));
  GS_CUDA(ctx, conv.alloc(w.Bpad, s));
  GS_CUDA(ctx, stag.alloc(w.Bpad, s));
  GS_CUDA(ctx, final_sweep.alloc(w.Bpad, s));
  GS_CUDA(ctx, errv.alloc(w.Bpad, s));
  GS_CUDA(ctx, cudaMemsetAsync(iters.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(conv.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(stag.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(final_sweep.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(V[0].get(), 0, len * sizeof(double), s));
  GS_CUDA(ctx, cudaMemsetAsync(W.get(), 0, len * sizeof(double), s));
  {
    std::vector<int> act(w.Bpad, 0);
    for (int p = 0; p < P; ++p) act[p] = 1;
    GS_CUDA(ctx, cudaMemcpyAsync(w.active.get(), act.data(), w.Bpad * sizeof(int), cudaMemcpyHostToDevice, s));
  }
  {
    std::vector<double> inf(w.Bpad, INFINITY);
    GS_CUDA(ctx, cudaMemcpyAsync(errv.get(), inf.data(), w.Bpad * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  gs_launch_begin(ctx, 1);
  k_pack<<<grid_for((int64_t)len), kThreads, 0, s>>>(dmu, M.get(), n, P, w.GW, w.G, 0.0, f->order);
  k_pack<<<grid_for((int64_t)len), kThreads, 0, s>>>(dnu, N.get(), n, P, w.GW, w.G, 0.0, f->order);
  k_sk_init<<<grid_for((int64_t)len), kThreads, 0, s>>>(da, w.T[0].get(), n, w.GW, w.G, P, w.cmax.get());
  gs_launch_end(ctx, 1);
  run_finalize(ctx, w, 0, 1, 0, ERRC_KERNEL_NOT_POSITIVE + 1, true);  // threshold of the first apply
  const int knp = ERRC_KERNEL_NOT_POSITIVE + 1;
  // ---- phi = H(a * 1) (transport.cpp:176) ------------------------------------------------------
  int a0 = run_apply(ctx, f, w, 0, MODE_SK_PHI, da, M.get(), V[0].get(), V[1].get(), true, true);
  run_finalize(ctx, w, 1, 1, 0, knp, true);
  // ---- sweeps (transport.cpp:177-227) ------------------------------------------------------------
  gs_status* hst = ctx->h_status;
  cudaEvent_t ev[2];
  cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
  bool ev_used[2] = {false, false};
  CtlArgs C{};
  C.active = w.active.get();
  C.gactive = w.gactive.get();
  C.GW = w.GW;
  C.errcol = w.errcol.get();
  C.iters = iters.get();
  C.conv = conv.get();
  C.stag = stag.get();
  C.final_sweep = final_sweep.get();
  C.err_out = errv.get();
  C.status = w.status.get();
  C.P = P;
  C.max_iter = max_iter;
  C.no_abort = (flags & GS_FLAG_NO_STAGNATION_ABORT) ? 1 : 0;
  C.tol = tol;
  for (int sweep = 1; sweep <= max_iter; ++sweep) {
    if (sweep >= 3) {
      const int slot = (sweep - 2) & 1;
      cudaEventSynchronize(ev[slot]);
      const gs_status st = hst[slot];
      if (st.error || st.n_active == 0) break;
    }
    // psi = H(a * V_s); W_s = N / max(psi, floor); T_0 = a * W_s
    a0 = run_apply(ctx, f, w, a0, MODE_SK_PSI, da, N.get(), nullptr, W.get(), true, true);
    run_finalize(ctx, w, 1, 1, 0, knp, true);
    // phi = H(a * W_s); err; V_{s+1} = M / max(phi, floor); T_0 = a * V_{s+1}
    a0 = run_apply(ctx, f, w, a0, MODE_SK_PHI, da, M.get(), V[sweep & 1].get(),
                   V[(sweep + 1) & 1].get(), true, true);
    run_finalize(ctx, w, 1, 1, 1, knp, true);
    C.sweep = sweep;
    gs_launch_begin(ctx, 1);
    k_sk_control<<<1, 1, 0, s>>>(C);
    gs_launch_end(ctx, 1);
    const int slot = sweep & 1;
    cudaMemcpyAsync(&hst[slot], w.status.get(), sizeof(gs_status), cudaMemcpyDeviceToHost, s);
    cudaEventRecord(ev[slot], s);
    ev_used[slot] = true;
  }
  (void)ev_used;
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  gs_status st;
  GS_CUDA(ctx, cudaMemcpy(&st, w.status.get(), sizeof st, cudaMemcpyDeviceToHost));
  if (st.error) {
    if (st.error == ERRC_DISCONNECTED + 1) {
      if (fail_pair) *fail_pair = st.fail_pair;
      if (fail_sweep) *fail_sweep = st.fail_sweep;
      if (flags & GS_FLAG_SINGLE)
        return gs_fail(ctx, ERRC_DISCONNECTED,
                       "marginal error stagnated above 0.5; are mu and nu in the same graph component?");
      return gs_fail(ctx, ERRC_DISCONNECTED,
                     "marginal error stagnated above 0.5 for pair " + std::to_string(st.fail_pair));
    }
    return gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, kKnpTransport);
  }
  // ---- cost / KL + outputs ------------------------------------------------------------------------
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  DevBuf<double> part, dcost, dkl;
  GS_CUDA(ctx, part.alloc((size_t)nchunks * P * 4, s));
  GS_CUDA(ctx, dcost.alloc(P, s));
  GS_CUDA(ctx, dkl.alloc(P, s));
  gs_launch_begin(ctx, 1);
  k_sk_cost_partial<<<dim3((unsigned)nchunks, P), kThreads, 0, s>>>(
      da, M.get(), N.get(), V[0].get(), V[1].get(), W.get(), final_sweep.get(), n, w.GW,
      part.get(), P);
  k_sk_cost_final<<<(P + 63) / 64, 64, 0, s>>>(part.get(), nchunks, P, 4.0 * f->t, dcost.get(), dkl.get());
  gs_launch_end(ctx, 1);
  DevBuf<double> ov, ow;
  double* dv = out_v;
  double* dw = out_w;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, ov.alloc((size_t)P * n, s));
    GS_CUDA(ctx, ow.alloc((size_t)P * n, s));
    dv = ov.get();
    dw = ow.get();
  }
  if (out_v) {
    gs_launch_begin(ctx, 1);
    k_unpack<<<grid_for((int64_t)P * n), kThreads, 0, s>>>(V[0].get(), dv, n, P, w.GW, V[1].get(), final_sweep.get(), f->newpos);
    gs_launch_end(ctx, 1);
    if (mem != GS_MEM_DEVICE) GS_TRY(finish_out(ctx, ov, out_v, (size_t)P * n, mem));
  }
  if (out_w) {
    gs_launch_begin(ctx, 1);
    k_unpack<<<grid_for((int64_t)P * n), kThreads, 0, s>>>(W.get(), dw, n, P, w.GW, nullptr, nullptr, f->newpos);
    gs_launch_end(ctx, 1);
    if (mem != GS_MEM_DEVICE) GS_TRY(finish_out(ctx, ow, out_w, (size_t)P * n, mem));
  }
  auto out_small = [&](void* dst, const void* src, size_t bytes) -> int {
    if (!dst) return GS_OK;
    GS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes,
                                 mem == GS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    return GS_OK;
  };
  GS_TRY(out_small(out_cost, dcost.get(), P * sizeof(double)));
  GS_TRY(out_small(out_kl, dkl.get(), P * sizeof(double)));
  GS_TRY(out_small(out_iters, iters.get(), P * sizeof(int)));
  GS_TRY(out_small(out_conv, conv.get(), P * sizeof(int)));
  GS_TRY(out_small(out_err, errv.get(), P * sizeof(double)));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// ============================================================================================
// Barycenter (barycenter.cpp:45-107)
// ============================================================================================
extern "C" int gs_barycenter(gs_ctx* ctx, const gs_filter* f, const double* a,
                             const double* members, int m, const double* alphas, int max_iter,
                             double tol, int mem, const gs_comm* comm, double* out_bary,
                             double* out_V, double* out_W, int* out_iters, int* out_conv,
                             double* out_err) {
  const int n = f->scaled->n;
  cudaStream_t s = ctx->stream;
  if (m < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "family must be non-empty");
  DevBuf<double> bmem, ba;
  const double *dmem, *da;
  GS_TRY(stage_in(ctx, bmem, members, (size_t)m * n, mem, &dmem));
  GS_TRY(stage_in(ctx, ba, a, (size_t)n, mem, &da));
  // family.validate (barycenter.cpp:32-43)
  {
    std::vector<double> sm;
    std::vector<int> fm, gm;
    GS_TRY(validate_columns(ctx, dmem, n, m, sm, fm, gm));
    for (int c = 0; c < m; ++c) GS_TRY(check_distribution(ctx, n, sm[c], fm[c], gm[c]));
  }
  std::vector<double> al(m);
  if (alphas) {
    if (mem == GS_MEM_DEVICE) {
      GS_CUDA(ctx, cudaMemcpy(al.data(), alphas, m * sizeof(double), cudaMemcpyDeviceToHost));
    } else {
      memcpy(al.data(), alphas, m * sizeof(double));
    }
  } else {
    for (int c = 0; c < m; ++c) al[c] = 1.0 / (double)m;
  }
  {
    double asum = 0.0;
    for (int c = 0; c < m; ++c) {
      if (!(al[c] >= 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "alphas must be non-negative");
      asum += al[c];
    }
    if (!comm && !(std::fabs(asum - 1.0) <= 1e-9)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "alphas must sum to 1");
  }
  GS_TRY(check_weights(ctx, da, n));
  if (!(tol > 0.0 && max_iter >= 1)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "bad parameters");
  DevBuf<double> aperm;
  GS_CUDA(ctx, aperm.alloc(n, s));
  gs_launch_begin(ctx, 1);
  k_gather<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(da, f->order, n, aperm.get());
  gs_launch_end(ctx, 1);
  da = aperm.get();

  Work w;
  GS_TRY(w.init(ctx, n, m, true, f));
  const size_t len = (size_t)w.Bpad * n;
  DevBuf<double> Mb, V[2], W, lb, bary, part, mass, dal, errbuf, derr;
  DevBuf<unsigned long long> lbmax;
  DevBuf<int> diters, dconv;
  GS_CUDA(ctx, Mb.alloc(len, s));
  GS_CUDA(ctx, V[0].alloc(len, s));
  GS_CUDA(ctx, V[1].alloc(len, s));
  GS_CUDA(ctx, W.alloc(len, s));
  GS_CUDA(ctx, lb.alloc(n, s));
  GS_CUDA(ctx, bary.alloc(n, s));
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  GS_CUDA(ctx, part.alloc(nchunks, s));
  GS_CUDA(ctx, mass.alloc(1, s));
  GS_CUDA(ctx, dal.alloc(m, s));
  GS_CUDA(ctx, errbuf.alloc(1, s));
  GS_CUDA(ctx, derr.alloc(1, s));
  GS_CUDA(ctx, lbmax.alloc(1, s));
  GS_CUDA(ctx, diters.alloc(1, s));
  GS_CUDA(ctx, dconv.alloc(1, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dal.get(), al.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemsetAsync(V[0].get(), 0, len * sizeof(double), s));
  GS_CUDA(ctx, cudaMemsetAsync(diters.get(), 0, sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(dconv.get(), 0, sizeof(int), s));
  {
    const double inf = INFINITY;
    GS_CUDA(ctx, cudaMemcpyAsync(derr.get(), &inf, sizeof(double), cudaMemcpyHostToDevice, s));
    cudaStreamSynchronize(s);
  }
  gs_launch_begin(ctx, 1);
  k_fill<<<grid_for(n), kThreads, 0, s>>>(bary.get(), n, 1.0 / n);
  k_pack<<<grid_for((int64_t)len), kThreads, 0, s>>>(dmem, Mb.get(), n, m, w.GW, w.G, 0.0, f->order);
  k_sk_init<<<grid_for((int64_t)len), kThreads, 0, s>>>(da, w.T[0].get(), n, w.GW, w.G, m, w.cmax.get());
  gs_launch_end(ctx, 1);
  run_finalize(ctx, w, 0, 1, 0, 0, false);
  const int knp = ERRC_KERNEL_NOT_POSITIVE + 1;
  // phi = H(a * 1) (barycenter.cpp:68); V_1 = M / max(phi, floor) in the epilogue
  int a0 = run_apply(ctx, f, w, 0, MODE_SK_PHI, da, Mb.get(), V[0].get(), V[1].get(), false, true);
  run_finalize(ctx, w, 1, 1, 0, knp, false);
  gs_status* hst = ctx->h_status;
  cudaEvent_t ev[2];
  cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
  int hook_rc = 0;
  for (int sweep = 1; sweep <= max_iter; ++sweep) {
    if (sweep >= 3) {
      const int slot = (sweep - 2) & 1;
      cudaEventSynchronize(ev[slot]);
      const gs_status st = hst[slot];
      if (st.error || st.done) break;
    }
    // psi = H(a * V) (barycenter.cpp:71)
    a0 = run_apply(ctx, f, w, a0, MODE_BARY_PSI, da, nullptr, nullptr, nullptr, false, true);
    run_finalize(ctx, w, 1, 0, 0, knp, false);
    // log-domain geometric mean (barycenter.cpp:75-82)
    gs_launch_begin(ctx, 1);
    k_bary_lb<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(w.acc.get(), dal.get(), n, m, w.GW, lb.get(), w.status.get());
    gs_launch_end(ctx, 1);
    if (comm && comm->allreduce) {
      hook_rc = comm->allreduce(comm->user, lb.get(), n, 0, (void*)s);
      if (hook_rc) break;
    }
    GS_CUDA(ctx, cudaMemsetAsync(lbmax.get(), 0, sizeof(unsigned long long), s));
    gs_launch_begin(ctx, 1);
    k_max_key<<<grid_for(n), kThreads, 0, s>>>(lb.get(), n, lbmax.get());
    k_bary_exp<<<(unsigned)nchunks, kThreads, 0, s>>>(lb.get(), lbmax.get(), n, bary.get(), part.get(), w.status.get());
    k_fold<<<1, kThreads, 0, s>>>(part.get(), nchunks, mass.get());
    k_bary_mass_check<<<1, 1, 0, s>>>(mass.get(), w.status.get());
    // W = bary / max(psi, floor); T_0 = a * W (barycenter.cpp:84-85)
    k_bary_w<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(
        bary.get(), mass.get(), w.acc.get(), da, n, m, w.GW, W.get(), w.T[a0].get(),
        w.cmax.get(), w.status.get());
    gs_launch_end(ctx, 1);
    run_finalize(ctx, w, 0, 1, 0, knp, false);
    // phi = H(a * W); err; V' = M / max(phi, floor) (barycenter.cpp:85-86, 70)
    a0 = run_apply(ctx, f, w, a0, MODE_SK_PHI, da, Mb.get(), V[sweep & 1].get(),
                   V[(sweep + 1) & 1].get(), false, true);
    run_finalize(ctx, w, 1, 1, 1, knp, false);
    gs_launch_begin(ctx, 1);
    k_bary_errlocal<<<1, 1, 0, s>>>(w.errcol.get(), m, errbuf.get());
    gs_launch_end(ctx, 1);
    if (comm && comm->allreduce) {
      hook_rc = comm->allreduce(comm->user, errbuf.get(), 1, 1, (void*)s);
      if (hook_rc) break;
    }
    gs_launch_begin(ctx, 1);
    k_bary_control<<<1, 1, 0, s>>>(errbuf.get(), w.status.get(), sweep, tol, diters.get(),
                                   dconv.get(), derr.get(), max_iter);
    gs_launch_end(ctx, 1);
    const int slot = sweep & 1;
    cudaMemcpyAsync(&hst[slot], w.status.get(), sizeof(gs_status), cudaMemcpyDeviceToHost, s);
    cudaEventRecord(ev[slot], s);
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (hook_rc) {
    ctx->err = "NcclError: allreduce hook failed";
    return GS_ERR_NCCL;
  }
  gs_status st;
  GS_CUDA(ctx, cudaMemcpy(&st, w.status.get(), sizeof st, cudaMemcpyDeviceToHost));
  if (st.error) {
    if (st.error == 1000 + ERRC_KERNEL_NOT_POSITIVE + 1)
      return gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, "barycenter iterate collapsed to zero");
    return gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, kKnpBary);
  }
  int h_iters = 0;
  GS_CUDA(ctx, cudaMemcpy(&h_iters, diters.get(), sizeof(int), cudaMemcpyDeviceToHost));
  // bary /= sum (barycenter.cpp:94), then Distribution::from_weights divides twice more
  // (transport.cpp:86-94); every sum is the deterministic DET-chunk fold.
  for (int pass = 0; pass < 3; ++pass) {
    gs_launch_begin(ctx, 1);
    k_chunk_sum<<<(unsigned)nchunks, kThreads, 0, s>>>(bary.get(), n, part.get());
    k_fold<<<1, kThreads, 0, s>>>(part.get(), nchunks, mass.get());
    k_scale_div<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(bary.get(), mass.get(), n);
    gs_launch_end(ctx, 1);
  }
  {
    DevBuf<double> bu;
    GS_CUDA(ctx, bu.alloc(n, s));
    gs_launch_begin(ctx, 1);
    k_gather<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(bary.get(), f->newpos, n, bu.get());
    gs_launch_end(ctx, 1);
    GS_TRY(gs_copy_out(ctx, out_bary, bu.get(), (size_t)n * sizeof(double), mem));
  }
  // final V lives in V[iters & 1] (V_s of the last sweep), W is single-buffered
  DevBuf<int> sel;
  GS_CUDA(ctx, sel.alloc(m, s));
  {
    std::vector<int> hs(m, h_iters);
    GS_CUDA(ctx, cudaMemcpyAsync(sel.get(), hs.data(), m * sizeof(int), cudaMemcpyHostToDevice, s));
  }
  DevBuf<double> ov, ow;
  double* dv = out_V;
  double* dw = out_W;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, ov.alloc((size_t)m * n, s));
    GS_CUDA(ctx, ow.alloc((size_t)m * n, s));
    dv = ov.get();
    dw = ow.get();
  }
  if (out_V) {
    gs_launch_begin(ctx, 1);
    k_unpack<<<grid_for((int64_t)m * n), kThreads, 0, s>>>(V[0].get(), dv, n, m, w.GW, V[1].get(), sel.get(), f->newpos);
    gs_launch_end(ctx, 1);
    if (mem != GS_MEM_DEVICE) GS_TRY(finish_out(ctx, ov, out_V, (size_t)m * n, mem));
  }
  if (out_W) {
    gs_launch_begin(ctx, 1);
    k_unpack<<<grid_for((int64_t)m * n), kThreads, 0, s>>>(W.get(), dw, n, m, w.GW, nullptr, nullptr, f->newpos);
    gs_launch_end(ctx, 1);
    if (mem != GS_MEM_DEVICE) GS_TRY(finish_out(ctx, ow, out_W, (size_t)m * n, mem));
  }
  int h_conv = 0;
  double h_err = 0.0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h_conv, dconv.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(&h_err, derr.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (out_iters) *out_iters = h_iters;
  if (out_conv) *out_conv = h_conv;
  if (out_err) *out_err = h_err;
  return GS_OK;
}

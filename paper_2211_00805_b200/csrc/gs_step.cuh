// gs_step.cuh -- the fused Chebyshev step kernel, templated on the scalar type S (double: the
// reference-exact path; float: the optional fp32 mode).
//
// Reference path: HeatFilter::apply (proj/src/heat.cpp:116-131) over
// SparseSymMatrix::multiply (proj/src/sparse.cpp:85-99), called twice per sweep by sinkhorn_many
// (proj/src/transport.cpp:144-239) and sinkhorn_barycenter (proj/src/barycenter.cpp:45-99).
//
// Layout ("grouped row-major"): a block of B vertex signals is G = B/GW column groups, each an
// n x GW row-major array (GW <= 64). A row segment of GW*sizeof(S) bytes is read by LPR lanes with
// 16-byte vector loads; a warp covers 32/LPR rows. A CTA covers RPC consecutive blocks of
// (8 warps x rows-per-warp) rows of one group, so neighbouring gathers share L1 lines (the
// vertices are in Cuthill-McKee order, gs_reorder.cu).
//
// One step k >= 2 (heat.cpp:124-130), per row i and column:
//     y   = sum_p vals[p] * T_{k-1}[cols[p]]        (fma chain from +0, CSR order)
//     T_k = 2 * (y - T_{k-1}[i]) - T_{k-2}[i]        (T_k overwrites T_{k-2} in place)
//     acc = fma(b_k, T_k, acc)
// Step 1: T_1 = y - T_0, acc = fma(b_1, T_1, (b_0/2) * T_0). The last step (k = K) does not store
// T_K; its epilogue consumes acc = p_K(L_s) x in registers:
//     SK_PSI  : psi -> colmin; W = N / max(psi, floor); next T_0 = a * W; colmax |T_0|
//     SK_PHI  : phi -> colmin; err += |V phi - M|; V' = M / max(phi, floor); next T_0 = a * V'
//     BARY_PSI: psi -> colmin and stored for the log-domain geometric mean.
// Column min/max are order-free (atomics on order-preserving keys of the double value); the L1
// error is accumulated in double through fixed-order per-CTA partials (deterministic).
//
// Per-layout choices (measured, profiles/r01c_summary.md): 512-byte fp64 rows (B = 64) one warp
// per row, gather batch 4, 48 registers / 5 CTAs, own rows staged by cp.async; 128/256-byte fp64
// rows (B = 16/32) batch 8, 64 registers / 4 CTAs; 64-byte narrow rows (B = 8) 8-byte lanes,
// 8 gathers, four row blocks per CTA; one row per lane (B <= 2 fp64 / 4 fp32) own rows loaded
// before the gathers, fp32 CSR read with aligned 16-byte loads; fp32 wide rows stage their own
// rows with per-warp TMA bulk copies. Round 2: one-row-per-lane layouts on several row blocks per
// CTA run k_cheb_lane below (per-warp CSR slices staged in shared memory by bulk copies, config 3:
// 607 -> 455 us per step); k_cheb_rec (16-byte records for the rows shared by several lanes) runs
// the 128-byte rows of graphs without index locality (config 4).
#pragma once

#include <cfloat>
#include <cstring>
#include <type_traits>

#include "gs_internal.cuh"

namespace gsk {

constexpr int kThreads = 256;
#ifndef GS_STEP_THREADS
#define GS_STEP_THREADS 256
#endif
constexpr int kStepThreads = GS_STEP_THREADS;  // threads of a k_cheb_step CTA
#ifndef GS_ROWS_PER_CTA
#define GS_ROWS_PER_CTA 4
#endif
constexpr int kRowsPerCta = GS_ROWS_PER_CTA;
#ifndef GS_ROWS_PER_CTA1
#define GS_ROWS_PER_CTA1 4
#endif
constexpr int kRowsPerCta1 = GS_ROWS_PER_CTA1;  // row blocks per CTA, one-row-per-lane layouts
#ifndef GS_GATHER_BATCH
#define GS_GATHER_BATCH 4
#endif
constexpr int kGatherBatch = GS_GATHER_BATCH;  // neighbour rows in flight per lane (wide fp64 rows)
#ifndef GS_GATHER_BATCH32
#define GS_GATHER_BATCH32 3
#endif
constexpr int kGatherBatch32 = GS_GATHER_BATCH32;  // wide fp32 rows (fewer registers -> 6 CTAs/SM)
#ifndef GS_GATHER_BATCH_MID
#define GS_GATHER_BATCH_MID 8
#endif
#ifndef GS_NARROW_GATHER_BATCH
#define GS_NARROW_GATHER_BATCH 8
#endif
#ifndef GS_PREFETCH_STAGES
#define GS_PREFETCH_STAGES 2
#endif
constexpr int kPrefetchStages = GS_PREFETCH_STAGES;

// CSR index prefetch (several lanes per row): the (col, val) chunk a row needs next is loaded
// while the current chunk's gathers are in flight -- the next LPR entries of the same row
// (GS_IDX_PREFETCH) and the first chunk of the warp's next row block (GS_ROW_PREFETCH), so the
// CSR stream's DRAM latency is not a link of the dependent index -> gather chain
#ifndef GS_IDX_PREFETCH
#define GS_IDX_PREFETCH 1
#endif
// one-row-per-lane layouts (own-row operands not staged by cp.async): load
// T_{k-1}[row], T_{k-2}[row] and acc[row] into registers before the gathers, so the streams'
// DRAM latency overlaps them instead of following them
#ifndef GS_EARLY_OWN
#define GS_EARLY_OWN 1
#endif
// one row per lane, fp32: a lane reads its row's columns and values four at a time with aligned
// 16-byte loads (carried across groups, the row's misalignment resolved by selects) instead of
// one 4-byte load per entry -- a quarter of the CSR load instructions (config 3: the LSU data
// pipe is 80% busy, two thirds of it on these per-lane scattered loads). Arrays carry kCsrPad.
#ifndef GS_CSR_VEC
#define GS_CSR_VEC 1
#endif
// cp.async-staged own rows: 1 = T_{k-1}, T_{k-2}, acc; 0 = T_{k-2} and acc only, T_{k-1}[row]
// read at the end of the row (an L1 hit: the row's diagonal entry has just gathered it)
#ifndef GS_PRE_TP
#define GS_PRE_TP 1
#endif
// 0: no shared-memory staging of the own rows; the wide layouts then load them into registers
// before the gathers (GS_EARLY_OWN)
#ifndef GS_WIDE_PREFETCH
#define GS_WIDE_PREFETCH 1
#endif
#ifndef GS_ROW_PREFETCH
#define GS_ROW_PREFETCH 0  // measured neutral-to-slower on config 1 (one chunk per row)
#endif
// own-row operands of the wide layouts staged by TMA bulk copies (one per warp and operand,
// completion on a per-warp mbarrier) instead of per-thread cp.async: the copies bypass the LSU
// data pipe, which the gathers and shuffles keep ~70% busy
// 0 = cp.async per thread, 1 = one bulk copy per warp, 2 = one per CTA row block (CTA barrier).
// Measured on config 1: fp64 128-130 us (cp.async) vs 152 (per warp) and 142 (per CTA); fp32
// mode 172 -> 189 sweeps/s with per-warp copies.
#ifndef GS_TMA_OWN64
#define GS_TMA_OWN64 0
#endif
#ifndef GS_TMA_OWN32
#define GS_TMA_OWN32 1
#endif

template <typename S>
struct RowIdx {  // a row's CSR range and this lane's entry of its first chunk (value as stored)
  int pb = 0, pe = 0, c = 0;
  S v = S(0);
};

enum StepMode { MODE_NONE = 0, MODE_SK_PSI = 1, MODE_SK_PHI = 2, MODE_BARY_PSI = 3 };

// ---- precision traits --------------------------------------------------------------------------
// S is the storage type of the Chebyshev vectors (T_{k-1}, T_{k-2}, acc, T_0) and of L_s's values;
// the arithmetic is fp64 in both modes (R = double).
//   double: the reference-exact path.
//   float : the optional 32-bit mode (DESIGN.md §4 "Precision"). A vector word is the upper half
//           of the fp64 word -- sign, the 11-bit fp64 exponent, 20 fraction bits -- rounded to
//           nearest, carried in a 4-byte `float` slot (bit pattern only, never used as IEEE
//           binary32). The reference's scaling vectors span more decades than binary32's 8-bit
//           exponent holds (config 1: per-column scaling with 66 decades of range still departs
//           from fp64 by sweep 20, profiles/r02_fp32_range.md); this word keeps fp64's range, so
//           the reference's 1e-300 floor and every control decision carry over, at 2^-21 relative
//           rounding per stored value. L_s's values are IEEE binary32 (entries of a scaled
//           Laplacian, no range issue).
template <typename S>
struct Prec;
template <>
struct Prec<double> {
  static constexpr double slack = 1e-12;   // positivity slack (transport.cpp:24,33)
  __device__ static __forceinline__ double dec(double x) { return x; }   // stored vector word
  __device__ static __forceinline__ double enc(double x) { return x; }
  __device__ static __forceinline__ double val(double v) { return v; }   // matrix value
  __device__ static __forceinline__ double fmat(double a, double b, double c) { return fma(a, b, c); }
};
template <>
struct Prec<float> {
  // rounding of the stored words (2^-21 relative each) accumulates over the K steps; the
  // positivity slack is 2^-14 of max |x| (the reference's 1e-12 assumes fp64 storage)
  static constexpr double slack = 0x1p-14;
  __device__ static __forceinline__ double dec(float w) { return __hiloint2double(__float_as_int(w), 0); }
  __device__ static __forceinline__ float enc(double x) {
    // round to nearest on the dropped 32 bits (the carry propagates into the exponent)
    const unsigned long long b = (unsigned long long)__double_as_longlong(x) + 0x80000000ull;
    return __int_as_float((int)(b >> 32));
  }
  __device__ static __forceinline__ double val(float v) { return (double)v; }
  __device__ static __forceinline__ double fmat(double a, double b, double c) { return fma(a, b, c); }
};

// bytes per lane for narrow rows (16 < GW * sizeof(S) <= 64): 8 gives more lanes per row, hence more
// (col, val) entries per coalesced index load and more gathers in flight per row
#ifndef GS_NARROW_VEC_BYTES
#define GS_NARROW_VEC_BYTES 8
#endif
#ifndef GS_NARROW_MAX_BYTES
#define GS_NARROW_MAX_BYTES 64  // widest row (GW * sizeof(S)) laid out as "narrow"
#endif
// bytes per lane for wide rows (GW * sizeof(S) > GS_NARROW_MAX_BYTES): 16 = one 512-byte fp64 row
// per warp; 32 or 64 put 2 or 4 rows in a warp, so one shuffle broadcasts (col, val) to all of
// them (measured slower for fp64 config 1: 164 vs 148 us)
#ifndef GS_WIDE_VEC_BYTES64
#define GS_WIDE_VEC_BYTES64 16
#endif
#ifndef GS_WIDE_VEC_BYTES32
#define GS_WIDE_VEC_BYTES32 16
#endif
template <int GW, typename S>
struct Lay {
  static constexpr bool NARROW = GW * (int)sizeof(S) <= GS_NARROW_MAX_BYTES && GW * (int)sizeof(S) > 16;
  static constexpr bool WIDE = GW * (int)sizeof(S) > GS_NARROW_MAX_BYTES;
  static constexpr int WVB = sizeof(S) == 8 ? GS_WIDE_VEC_BYTES64 : GS_WIDE_VEC_BYTES32;
  static constexpr int VB = NARROW ? GS_NARROW_VEC_BYTES : (WIDE ? WVB : 16);
  static constexpr int VEC = GW * (int)sizeof(S) >= VB ? (VB >= (int)sizeof(S) ? VB / (int)sizeof(S) : 1) : GW;
  static constexpr int LPR = GW / VEC;                 // lanes per row
  static constexpr int RPW = 32 / LPR;                 // rows per warp
  static constexpr int ROWS = (kStepThreads / 32) * RPW;  // rows per CTA block
  // gathers in flight per row: narrow rows have few registers per gather, so go deeper
  // wider lanes keep the bytes in flight per lane: batch scaled down by VB / 16
  static constexpr int GBW0 = (sizeof(S) == 4 ? kGatherBatch32 : kGatherBatch) * 16 / (VB > 16 ? VB : 16);
  // fp64 rows wider than a narrow row but shorter than a warp (B = 16 / 32: 128 / 256 bytes,
  // config 4): a whole chunk's gathers in flight, fewer CTAs (GS_*_MID)
  static constexpr bool MID = WIDE && LPR < 32 && sizeof(S) == 8;
  static constexpr int GB = NARROW ? (GS_NARROW_GATHER_BATCH < LPR ? GS_NARROW_GATHER_BATCH : LPR)
                                   : MID ? (GS_GATHER_BATCH_MID < LPR ? GS_GATHER_BATCH_MID : LPR)
                                         : (GBW0 < 1 ? 1 : GBW0);
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

// 16/8/4-byte vector moves between memory and a register array (explicit components, so the
// array stays in registers)
template <typename S, int VEC, bool RO>
__device__ __forceinline__ void ld_vec_impl(const S* p, S (&v)[VEC]) {
  if constexpr (VEC * sizeof(S) > 16) {  // several 16-byte chunks
    constexpr int C = 16 / (int)sizeof(S);
#pragma unroll
    for (int h = 0; h < VEC / C; ++h) {
      S t[C];
      ld_vec_impl<S, C, RO>(p + h * C, t);
#pragma unroll
      for (int e = 0; e < C; ++e) v[h * C + e] = t[e];
    }
  } else if constexpr (std::is_same<S, double>::value && VEC == 2) {
    const double2 t = RO ? __ldg(reinterpret_cast<const double2*>(p)) : *reinterpret_cast<const double2*>(p);
    v[0] = t.x;
    v[1] = t.y;
  } else if constexpr (std::is_same<S, float>::value && VEC == 4) {
    const float4 t = RO ? __ldg(reinterpret_cast<const float4*>(p)) : *reinterpret_cast<const float4*>(p);
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
  } else if constexpr (std::is_same<S, float>::value && VEC == 2) {
    const float2 t = RO ? __ldg(reinterpret_cast<const float2*>(p)) : *reinterpret_cast<const float2*>(p);
    v[0] = t.x;
    v[1] = t.y;
  } else {
    static_assert(VEC == 1, "vector width");
    v[0] = RO ? __ldg(p) : *p;
  }
}
template <typename S, int VEC>
__device__ __forceinline__ void ld_vec(const S* p, S (&v)[VEC]) {  // read-only path
  ld_vec_impl<S, VEC, true>(p, v);
}
template <typename S, int VEC>
__device__ __forceinline__ void ld_vec_rw(const S* p, S (&v)[VEC]) {
  ld_vec_impl<S, VEC, false>(p, v);
}
template <typename S, int VEC>
__device__ __forceinline__ void st_vec(S* p, const S (&v)[VEC]) {
  if constexpr (VEC * sizeof(S) > 16) {
    constexpr int C = 16 / (int)sizeof(S);
#pragma unroll
    for (int h = 0; h < VEC / C; ++h) {
      S t[C];
#pragma unroll
      for (int e = 0; e < C; ++e) t[e] = v[h * C + e];
      st_vec<S, C>(p + h * C, t);
    }
  } else if constexpr (std::is_same<S, double>::value && VEC == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  } else if constexpr (std::is_same<S, float>::value && VEC == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (std::is_same<S, float>::value && VEC == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

// CSR entry loads (read-only path)
template <typename T>
__device__ __forceinline__ T ld_idx(const T* p) {
  return __ldg(p);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

struct ColState {  // per column (Bpad entries each)
  int* active;               // nullable
  int* gactive;              // active columns per group (nullable)
  unsigned long long* cmin;  // min of the apply output
  unsigned long long* cmax;  // max |next T_0|
  double* thr;               // positivity threshold of the current apply
  double* errcol;            // L1 marginal error
  double* part_err;          // [tiles][Bpad]
};

struct StepArgs {  // vector pointers are S* of the launch's precision
  const int* __restrict__ offs;
  const int* __restrict__ cols;
  const void* vals;
  int n, tiles, g0, Gl, Bpad;  // rows [row0, n) in `tiles` CTA tiles per column group
  int row0, tile0;             // first row; index of the first tile in the error partials
  int warp_rows;               // one warp per row (k_cheb_step_w1; one-column fp64 problems)
  int tile_period;             // > 1: CTA b runs tile tile_of(b) -- every window's heaviest tile first
  int lane;                    // one row per lane: the staged kernel k_cheb_lane (offs / cols / vals may be
                               // its odd-stride copy, gs_lane.cu: pad entries have column -1)
  int64_t ld;         // rows per column group (n, or local + halo rows for a row partition)
  const void* Tprev;  // T_{k-1}
  void* Tout;         // T_{k-2} in, T_k out (or next T_0 / SpMM output)
  void* acc;
  double bk, b0h;
  int k;              // 0 = plain SpMM into Tout
  // deferred accumulation: acc += b_j T_j is applied for up to three steps at once (the own rows
  // T_{k-2}, T_{k-1}, T_k are all at hand in step k), oldest term first -- the same fma chain
  // as one update per step, with a third of the acc traffic (host schedule: acc_schedule)
  int acc_terms;      // 0 = defer; 1..3 = add b_{k-j+1..k} T_{k-j+1..k}
  int acc_init;       // 1 = no acc yet: start from (b_0 / 2) T_0 (T_0 = own row of T_{k-1} or T_{k-2})
  int store_t;        // 0 = T_k is never read again (last step)
  double bk1, bk2;    // b_{k-1}, b_{k-2}
  const gs_status* status;
  ColState cs;
  const void* recs;    // k_cheb_rec: the CSR entries as 16-byte records (gs_layout::recs); nullptr = off
  const int* rec_key;  // k_cheb_blk: 8-row block records (gs_layout::rec_key / rec_val)
  const void* rec_val;
  // fused epilogue operands: always fp64 (in the fp32 mode only the Chebyshev recurrence runs
  // in fp32; the scaling vectors keep the reference's fp64 range, DESIGN.md §4 "Precision")
  const double* a;      // n (epilogue)
  const double* M;      // PSI: N (targets); PHI: M (sources / members)
  const double* Vcur;   // PHI: V of this sweep
  double* Wout;         // PSI: W; PHI: V of the next sweep
  double* psi;          // BARY_PSI in the 32-bit mode: psi in fp64 (the fp64 mode uses acc)
  // BARY_PSI, one column group: the log-domain geometric mean fused into the epilogue
  // (barycenter.cpp:75-78): lb[row] = sum_c alphas[c] log(clamp(psi[row][c])) in member order,
  // and the max of lb over the grid in *lbmax (order-preserving key); nullptr = separate passes
  double* lb;
  const double* alphas;
  unsigned long long* lbmax;
  int m;
};

// Launch order of the tiles of a degree-sorted layout: with P = A.tile_period tiles per window,
// CTAs first run the heavier half of every window (tiles t with t mod P < P/2: the window's
// longest rows), then the lighter halves, so the tail wave of the grid is made of short tiles.
// The tile -> rows map (and with it every result and error partial) is unchanged.
__device__ __forceinline__ int tile_of(const StepArgs& A, int b) {
  const int P = A.tile_period;
  if (P <= 1) return b;
  const int H = P / 2, Lh = P - H;
  const int full = A.tiles / P, rem = A.tiles % P;
  const int heavy = full * H + min(rem, H);  // tiles in the heavier halves
  if (b < heavy) return b / H * P + b % H;
  b -= heavy;
  return b / Lh * P + H + b % Lh;
}

template <typename S, int GW, int MODE>
__device__ __forceinline__ void finish_row(const StepArgs& A, int g, int row, int q,
                                           const double (&y)[Lay<GW, S>::VEC],
                                           double (&mn)[Lay<GW, S>::VEC],
                                           double (&mx)[Lay<GW, S>::VEC],
                                           double (&er)[Lay<GW, S>::VEC], const S* pre,
                                           int pre_stride, bool pre_tp = true);

// encode + vector store of fp64 register values into storage words
template <typename S, int VEC>
__device__ __forceinline__ void st_enc(S* p, const double (&v)[VEC]) {
  S t[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) t[e] = Prec<S>::enc(v[e]);
  st_vec<S, VEC>(p, t);
}

// One row of one Chebyshev step; epilogue partials accumulate in mn/mx/er (double).
template <typename S, int GW, int MODE>
__device__ __forceinline__ void cheb_row(const StepArgs& A, int g, int row, int sub, int q,
                                         double (&mn)[Lay<GW, S>::VEC],
                                         double (&mx)[Lay<GW, S>::VEC],
                                         double (&er)[Lay<GW, S>::VEC], const S* pre,
                                         int pre_stride, const RowIdx<S>& ri, bool pre_tp = true) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC, LPR = L::LPR;
  using P = Prec<S>;
  const bool valid = row < A.n;
  const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
  const size_t idx = gbase + (size_t)(valid ? row : 0) * GW;
  const S* __restrict__ Tp = static_cast<const S*>(A.Tprev) + gbase;
  const S* __restrict__ vals = static_cast<const S*>(A.vals);
  S own[3 * VEC];  // early own-row operands (GS_EARLY_OWN): tp, t2, a0
  // layouts whose own rows k_cheb_step stages in shared memory never take the early path
  constexpr bool STAGED = GS_WIDE_PREFETCH && VEC * sizeof(S) >= 16 && (VEC * sizeof(S)) % 16 == 0;
  // measured: config 3 (one row per lane) 589 -> 564 us; config 2 (narrow rows) 341 -> 362 us
  constexpr bool EARLY = GS_EARLY_OWN && !STAGED && (LPR == 1 || !GS_WIDE_PREFETCH);
  const bool early = EARLY && !pre && valid && A.k != 0;
  if (EARLY && early) {
#pragma unroll
    for (int e = 0; e < 3 * VEC; ++e) own[e] = S(0);
    S t[VEC];
    ld_vec<S, VEC>(static_cast<const S*>(A.Tprev) + idx, t);
#pragma unroll
    for (int e = 0; e < VEC; ++e) own[e] = t[e];
    if (A.k >= 2) {
      ld_vec_rw<S, VEC>(static_cast<const S*>(A.Tout) + idx, t);
#pragma unroll
      for (int e = 0; e < VEC; ++e) own[VEC + e] = t[e];
    }
    if (A.acc_terms > 0 && !A.acc_init) {
      ld_vec_rw<S, VEC>(static_cast<const S*>(A.acc) + idx, t);
#pragma unroll
      for (int e = 0; e < VEC; ++e) own[2 * VEC + e] = t[e];
    }
  }
  // ---- y = L_s T_{k-1} (row), fp64 fma chain ----------------------------------------------------
  double y[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) y[e] = 0.0;
  if constexpr (LPR == 1) {
    if (valid) {
      int p = __ldg(A.offs + row);
      const int pe = __ldg(A.offs + row + 1);
      if constexpr (GS_CSR_VEC && sizeof(S) == 4) {
        const int off = p & 3;
        const int* cbase = A.cols + (p - off);
        const float* vbase = reinterpret_cast<const float*>(vals) + (p - off);
        int4 ca = __ldg(reinterpret_cast<const int4*>(cbase));
        float4 va = __ldg(reinterpret_cast<const float4*>(vbase));
        // element u of the group starting at p: block a (u + off < 4) or the next block b
        auto sel_i = [&](const int4& a, const int4& b, int k) {  // k = u + off in 0..6
          return k == 0 ? a.x : k == 1 ? a.y : k == 2 ? a.z : k == 3 ? a.w : k == 4 ? b.x : k == 5 ? b.y : b.z;
        };
        auto sel_f = [&](const float4& a, const float4& b, int k) {
          return k == 0 ? a.x : k == 1 ? a.y : k == 2 ? a.z : k == 3 ? a.w : k == 4 ? b.x : k == 5 ? b.y : b.z;
        };
        for (int blk = 1; p + 4 <= pe; p += 4, ++blk) {
          const int4 cb = __ldg(reinterpret_cast<const int4*>(cbase) + blk);
          const float4 vb = __ldg(reinterpret_cast<const float4*>(vbase) + blk);
          int cc[4];
          S vv[4];
          S xx[4][VEC];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            cc[u] = sel_i(ca, cb, u + off);
            vv[u] = sel_f(va, vb, u + off);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) ld_vec<S, VEC>(Tp + (size_t)cc[u] * GW, xx[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(vv[u]), P::dec(xx[u][e]), y[e]);
          ca = cb;
          va = vb;
        }
      }
      for (; p + 4 <= pe; p += 4) {
        int cc[4];
        S vv[4];
        S xx[4][VEC];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cc[u] = __ldg(A.cols + p + u);
          vv[u] = __ldg(vals + p + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) ld_vec<S, VEC>(Tp + (size_t)cc[u] * GW, xx[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(vv[u]), P::dec(xx[u][e]), y[e]);
      }
      for (; p < pe; ++p) {
        const int c = __ldg(A.cols + p);
        const S v = __ldg(vals + p);
        S x[VEC];
        ld_vec<S, VEC>(Tp + (size_t)c * GW, x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(v), P::dec(x[e]), y[e]);
      }
    }
  } else {
    // the LPR lanes of a row load LPR consecutive (col, val) entries with one coalesced access
    // and broadcast them by shuffle; the fma chain still runs in CSR order.
    const int sub_lane0 = sub * LPR;
    const unsigned mask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << sub_lane0);
    const int pb = ri.pb, pe = ri.pe;  // first chunk loaded by the caller (k_cheb_step)
    constexpr int GB = L::GB;
    int myc = ri.c;
    S myv = ri.v;
    for (int p0 = pb; p0 < pe; p0 += LPR) {
      int nxc = 0;
      S nxv = S(0);
      if constexpr (GS_IDX_PREFETCH) {
        if (p0 + LPR + q < pe) {
          nxc = ld_idx(A.cols + p0 + LPR + q);
          nxv = ld_idx(vals + p0 + LPR + q);
        }
      } else if (p0 > pb) {
        myc = 0;
        myv = S(0);
        if (p0 + q < pe) {
          myc = ld_idx(A.cols + p0 + q);
          myv = ld_idx(vals + p0 + q);
        }
      }
      const int cnt = min(LPR, pe - p0);
      int u = 0;
      for (; u + GB <= cnt; u += GB) {
        int cc[GB];
        S vv[GB];
        S xx[GB][VEC];
#pragma unroll
        for (int j = 0; j < GB; ++j) {
          cc[j] = __shfl_sync(mask, myc, u + j, LPR);
          vv[j] = __shfl_sync(mask, myv, u + j, LPR);
        }
#pragma unroll
        for (int j = 0; j < GB; ++j) ld_vec<S, VEC>(Tp + (size_t)cc[j] * GW, xx[j]);
#pragma unroll
        for (int j = 0; j < GB; ++j)
#pragma unroll
          for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(vv[j]), P::dec(xx[j][e]), y[e]);
      }
      for (; u < cnt; ++u) {
        const int c = __shfl_sync(mask, myc, u, LPR);
        const S v = __shfl_sync(mask, myv, u, LPR);
        S x[VEC];
        ld_vec<S, VEC>(Tp + (size_t)c * GW, x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(v), P::dec(x[e]), y[e]);
      }
      if constexpr (GS_IDX_PREFETCH) {
        myc = nxc;
        myv = nxv;
      }
    }
  }
  if (!valid) return;
  if (EARLY && early) finish_row<S, GW, MODE>(A, g, row, q, y, mn, mx, er, own, VEC);
  else finish_row<S, GW, MODE>(A, g, row, q, y, mn, mx, er, pre, pre_stride, pre_tp);
}

// The rest of a row's step once y = (L_s T_{k-1})[row] is known: the recurrence, the deferred
// acc update and the stores / fused epilogue (row < A.n).
template <typename S, int GW, int MODE>
__device__ __forceinline__ void finish_row_ops(const StepArgs& A, int g, int row, int q,
                                               const double (&y)[Lay<GW, S>::VEC],
                                               double (&mn)[Lay<GW, S>::VEC],
                                               double (&mx)[Lay<GW, S>::VEC],
                                               double (&er)[Lay<GW, S>::VEC],
                                               const S (&tps)[Lay<GW, S>::VEC],
                                               const S (&t2s)[Lay<GW, S>::VEC],
                                               const S (&a0s)[Lay<GW, S>::VEC],
                                               const double* epi = nullptr);

template <typename S, int GW, int MODE>
__device__ __forceinline__ void finish_row(const StepArgs& A, int g, int row, int q,
                                           const double (&y)[Lay<GW, S>::VEC],
                                           double (&mn)[Lay<GW, S>::VEC],
                                           double (&mx)[Lay<GW, S>::VEC],
                                           double (&er)[Lay<GW, S>::VEC], const S* pre,
                                           int pre_stride, bool pre_tp) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC;
  const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
  const size_t idx = gbase + (size_t)row * GW;
  if (A.k == 0) {  // plain SpMM (sparse.cpp:85-99)
    st_enc<S, VEC>(static_cast<S*>(A.Tout) + idx, y);
    return;
  }
  // ---- own-row operands (prefetched into shared memory by cp.async when `pre`) ---------------
  const bool read_acc = A.acc_terms > 0 && !A.acc_init;
  S tps[VEC], t2s[VEC], a0s[VEC];
  if (pre && pre_tp) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      tps[e] = pre[e];
      t2s[e] = pre[pre_stride + e];
      a0s[e] = pre[2 * pre_stride + e];
    }
  } else if (pre) {  // T_{k-2}, acc staged; T_{k-1}[row] read directly (L1-hot: just gathered)
    ld_vec<S, VEC>(static_cast<const S*>(A.Tprev) + idx, tps);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      t2s[e] = pre[e];
      a0s[e] = pre[pre_stride + e];
    }
  } else {
    ld_vec<S, VEC>(static_cast<const S*>(A.Tprev) + idx, tps);
    if (A.k >= 2) ld_vec_rw<S, VEC>(static_cast<const S*>(A.Tout) + idx, t2s);
    if (read_acc) ld_vec_rw<S, VEC>(static_cast<const S*>(A.acc) + idx, a0s);
  }
  finish_row_ops<S, GW, MODE>(A, g, row, q, y, mn, mx, er, tps, t2s, a0s);
}

// The recurrence, the deferred acc update and the stores / fused epilogue of one row, from its
// own-row operands T_{k-1}[row], T_{k-2}[row], acc[row] (storage words; k >= 1, row < A.n).
template <typename S, int GW, int MODE>
__device__ __forceinline__ void finish_row_ops(const StepArgs& A, int g, int row, int q,
                                               const double (&y)[Lay<GW, S>::VEC],
                                               double (&mn)[Lay<GW, S>::VEC],
                                               double (&mx)[Lay<GW, S>::VEC],
                                               double (&er)[Lay<GW, S>::VEC],
                                               const S (&tps)[Lay<GW, S>::VEC],
                                               const S (&t2s)[Lay<GW, S>::VEC],
                                               const S (&a0s)[Lay<GW, S>::VEC],
                                               const double* epi) {
  // epi (optional): the Sinkhorn epilogue's operands already in registers -- M[row] (VEC),
  // Vcur[row] (VEC, PHI only), a[row] -- loaded one row ahead by the caller (k_cheb_win)
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC;
  using P = Prec<S>;
  const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
  const size_t idx = gbase + (size_t)row * GW;
  double tp[VEC], t2[VEC], a0[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    tp[e] = P::dec(tps[e]);
    t2[e] = P::dec(t2s[e]);
    a0[e] = P::dec(a0s[e]);
  }
  // ---- recurrence (heat.cpp:121-130) ----------------------------------------------------------
  double t[VEC], ac[VEC];
  if (A.k == 1) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) t[e] = y[e] - tp[e];
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) t[e] = 2.0 * (y[e] - tp[e]) - t2[e];
  }
  // acc = fma(b_k, T_k, acc) for the pending steps, oldest first (heat.cpp:122,129)
  if (A.acc_terms > 0) {
    const double bk = A.bk, bk1 = A.bk1, bk2 = A.bk2, b0h = A.b0h;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      double base = A.acc_init ? b0h * (A.k == 1 ? tp[e] : t2[e]) : a0[e];
      if (A.acc_terms >= 3) base = P::fmat(bk2, t2[e], base);
      if (A.acc_terms >= 2) base = P::fmat(bk1, tp[e], base);
      ac[e] = P::fmat(bk, t[e], base);
    }
  }
  if constexpr (MODE == MODE_NONE) {
    if (A.store_t) st_enc<S, VEC>(static_cast<S*>(A.Tout) + idx, t);
    if (A.acc_terms > 0) st_enc<S, VEC>(static_cast<S*>(A.acc) + idx, ac);
  } else {
    // ---- fused epilogue of the last step (fp64; transport.cpp:171-184, barycenter.cpp:71) ----
    const int* act = A.cs.active;
    const int col0 = g * GW + q * VEC;
#pragma unroll
    for (int e = 0; e < VEC; ++e) mn[e] = fmin(mn[e], ac[e]);
    if constexpr (MODE == MODE_SK_PSI || MODE == MODE_SK_PHI) {
      double op1[VEC], nx[VEC], t0[VEC];
      if (epi) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) op1[e] = epi[e];
      } else {
        ld_vec<double, VEC>(A.M + idx, op1);
      }
      const double ai = epi ? epi[2 * VEC] : __ldg(A.a + row);
      if constexpr (MODE == MODE_SK_PHI) {
        double v[VEC];
        if (epi) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) v[e] = epi[VEC + e];
        } else {
          ld_vec_rw<double, VEC>(A.Vcur + idx, v);
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) er[e] = er[e] + fabs(v[e] * ac[e] - op1[e]);  // transport.cpp:184
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        nx[e] = op1[e] / fmax(ac[e], GS_FLOOR);  // W (transport.cpp:180) / V' (:178), kDivisionFloor
        t0[e] = ai * nx[e];                      // a .* x (transport.cpp:172)
        mx[e] = fmax(mx[e], fabs(t0[e]));
      }
      st_enc<S, VEC>(static_cast<S*>(A.Tout) + idx, t0);
      double* wo = A.Wout + idx;
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (!act || act[col0 + e]) wo[e] = nx[e];
    } else {  // MODE_BARY_PSI: psi kept in fp64 for the log-domain mean
      if constexpr (sizeof(S) == 4) st_vec<double, VEC>(A.psi + idx, ac);
      else st_vec<S, VEC>(static_cast<S*>(A.acc) + idx, ac);
      if (A.lb) {
        // fused log-domain geometric mean (barycenter.cpp:75-78; k_bary_lb's arithmetic): the
        // row's lanes hold its m <= GW columns; lane 0 of the row folds them in member order
        constexpr int LPR = L::LPR;
        const int lane = threadIdx.x & 31;
        const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (lane / LPR * LPR));
        double lg[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) lg[e] = log(fmin(fmax(ac[e], GS_FLOOR), GS_CEIL));
        double acc = 0.0;
        for (int c = 0; c < A.m; ++c) {
          double mine = lg[0];
#pragma unroll
          for (int e = 1; e < VEC; ++e)
            if (c % VEC == e) mine = lg[e];
          const double v = LPR == 1 ? mine : __shfl_sync(gmask, mine, c / VEC, LPR);
          acc = fma(A.alphas[c], v, acc);
        }
        if (q == 0) {
          A.lb[row] = acc;
          mx[0] = fmax(mx[0], acc);
        }
      }
    }
  }
}

// CTA-level fold of the epilogue partials: min/max by atomics on keys, error partial per tile.
template <typename S, int GW, int MODE, int NT = kStepThreads>
__device__ __forceinline__ void block_epilogue(const StepArgs& A, int g, int tile, int warp, int sub,
                                               int q, double (&mn)[Lay<GW, S>::VEC],
                                               double (&mx)[Lay<GW, S>::VEC],
                                               double (&er)[Lay<GW, S>::VEC]) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC, LPR = L::LPR;
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      mn[e] = fmin(mn[e], __shfl_xor_sync(0xffffffffu, mn[e], off));
      mx[e] = fmax(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], off));
      er[e] = er[e] + __shfl_xor_sync(0xffffffffu, er[e], off);
    }
  }
  __shared__ double s_mn[NT / 32][GW], s_mx[NT / 32][GW], s_er[NT / 32][GW];
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
    for (int w = 1; w < NT / 32; ++w) {
      a_mn = fmin(a_mn, s_mn[w][c]);
      a_mx = fmax(a_mx, s_mx[w][c]);
      a_er = a_er + s_er[w][c];
    }
    const int col = g * GW + c;
    atomicMin(A.cs.cmin + col, dkey(a_mn));
    if constexpr (MODE == MODE_SK_PSI || MODE == MODE_SK_PHI) atomicMax(A.cs.cmax + col, dkey(a_mx));
    if constexpr (MODE == MODE_BARY_PSI)
      if (A.lbmax && c == 0) atomicMax(A.lbmax, dkey(a_mx));  // max of the fused log-sum
    if constexpr (MODE == MODE_SK_PHI) A.cs.part_err[(size_t)tile * A.Bpad + col] = a_er;
  }
}

// A CTA owns RPC x (8 warps x rows-per-warp) consecutive rows of one column group. Own-row
// operands of the next row block (T_{k-1}[i], T_{k-2}[i], acc[i]) are copied to shared memory with
// cp.async while this block's neighbour gathers run (16-byte vector rows only).
// resident CTAs per SM the register allocation of the plain step must allow (0 = compiler's choice)
#ifndef GS_MIN_BLOCKS
#define GS_MIN_BLOCKS 5
#endif
#ifndef GS_MIN_BLOCKS_MID
#define GS_MIN_BLOCKS_MID 4  // config-4 shape at n = 1e6: 343 -> 319 us with GS_GATHER_BATCH_MID 8
#endif
#ifndef GS_MIN_BLOCKS_NARROW
#define GS_MIN_BLOCKS_NARROW 5
#endif
#ifndef GS_MIN_BLOCKS32
#define GS_MIN_BLOCKS32 5
#endif
template <typename S, int GW, int MODE, int RPC>
__global__ void __launch_bounds__(kStepThreads, MODE != MODE_NONE ? 0
                                                  : (Lay<GW, S>::NARROW ? GS_MIN_BLOCKS_NARROW
                                                     : Lay<GW, S>::MID ? GS_MIN_BLOCKS_MID
                                                     : (sizeof(S) == 4 ? GS_MIN_BLOCKS32 : GS_MIN_BLOCKS)))
    k_cheb_step(const StepArgs A) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC, LPR = L::LPR, RPW = L::RPW;
  constexpr int BLOCK_ROWS = (kStepThreads / 32) * RPW;
  constexpr bool PREFETCH = GS_WIDE_PREFETCH && VEC * sizeof(S) >= 16 && (VEC * sizeof(S)) % 16 == 0;
  constexpr int CH = (int)(VEC * sizeof(S) / 16);  // 16-byte cp.async chunks per operand
  if (A.status && (A.status->error || A.status->done)) return;
  const int tl = tile_of(A, blockIdx.x / A.Gl);
  const int tile = A.tile0 + tl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = MODE == MODE_BARY_PSI ? -INFINITY : 0.0;  // BARY_PSI: max of the fused log-sum
    er[e] = 0.0;
  }
  const int base = A.row0 + tl * (BLOCK_ROWS * RPC) + warp * RPW + sub;
  // CSR ranges of this lane group's RPC rows: lane q < RPC holds block q's (pb, pe)
  static_assert(LPR == 1 || LPR >= RPC, "one lane per row block holds its offsets");
  int o_pb = 0, o_pe = 0;
  if constexpr (LPR > 1) {
    const int r = base + q * BLOCK_ROWS;
    if (q < RPC && r < A.n) {
      o_pb = __ldg(A.offs + r);
      o_pe = __ldg(A.offs + r + 1);
    }
  }
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << (LPR & 31)) - 1u) << (sub * LPR));
  auto row_idx = [&](int j) {  // block j's range and this lane's first-chunk entry
    RowIdx<S> ri;
    if constexpr (LPR > 1) {
      ri.pb = __shfl_sync(gmask, o_pb, j, LPR);
      ri.pe = __shfl_sync(gmask, o_pe, j, LPR);
      if (ri.pb + q < ri.pe) {
        ri.c = ld_idx(A.cols + ri.pb + q);
        ri.v = ld_idx(static_cast<const S*>(A.vals) + ri.pb + q);
      }
    }
    return ri;
  };
  RowIdx<S> cur = row_idx(0);
  auto next_idx = [&](int j) {  // row j's index state, prefetched one row block ahead
    RowIdx<S> nx;
    if constexpr (GS_ROW_PREFETCH) {
      if (j + 1 < RPC) nx = row_idx(j + 1);
    }
    return nx;
  };
  if constexpr (PREFETCH) {
    constexpr int STG = kPrefetchStages;
    constexpr int PS = kStepThreads * VEC;  // elements per operand per stage
    constexpr int TMA_ = sizeof(S) == 8 ? GS_TMA_OWN64 : GS_TMA_OWN32;
    constexpr int NOPS = (GS_PRE_TP || TMA_ != 0) ? 3 : 2;  // staged operands per row
    __shared__ __align__(128) S s_pre[STG][NOPS][PS];
    const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
    auto issue = [&](int j) {
      const int row = base + j * BLOCK_ROWS;
      if (j < RPC && row < A.n && A.k != 0) {
        const size_t idx = gbase + (size_t)row * GW;
        S* d = &s_pre[j % STG][0][threadIdx.x * VEC];
        constexpr int CE = 16 / (int)sizeof(S);
#pragma unroll
        for (int h = 0; h < CH; ++h) {
          constexpr int O = GS_PRE_TP ? 1 : 0;  // operand slot of T_{k-2}
          if constexpr (GS_PRE_TP) cp_async16(d + h * CE, static_cast<const S*>(A.Tprev) + idx + h * CE);
          if (A.k >= 2) cp_async16(d + O * PS + h * CE, static_cast<const S*>(A.Tout) + idx + h * CE);
          if (A.acc_terms > 0 && !A.acc_init)
            cp_async16(d + (O + 1) * PS + h * CE, static_cast<const S*>(A.acc) + idx + h * CE);
        }
      }
      cp_async_commit();
    };
    constexpr int TMA = sizeof(S) == 8 ? GS_TMA_OWN64 : GS_TMA_OWN32;
    if constexpr (TMA != 0) {
      // warp w's RPW rows of block j are one contiguous RPW * GW * sizeof(S) byte run in global
      // memory and in s_pre (slot = thread * VEC); lane 0 copies it per operand
      // TMA == 2: the CTA's BLOCK_ROWS rows of block j, one copy per operand by thread 0
      constexpr int NB = TMA == 1 ? kStepThreads / 32 : 1;
      __shared__ __align__(8) unsigned long long s_bar[NB][STG];
      constexpr int WE = TMA == 1 ? RPW * GW : 0;  // elements per warp per operand
      constexpr int CR = TMA == 1 ? RPW : BLOCK_ROWS;  // rows per copy
      const int bw = TMA == 1 ? warp : 0;
      const bool issuer = TMA == 1 ? lane == 0 : threadIdx.x == 0;
      if (issuer) {
#pragma unroll
        for (int st = 0; st < STG; ++st) mbar_init(&s_bar[bw][st], 1);
        fence_proxy_async();
      }
      if constexpr (TMA == 1) __syncwarp(); else __syncthreads();
      const int wrow0 = TMA == 1 ? base - sub : A.row0 + tl * (BLOCK_ROWS * RPC);  // first row, block 0
      auto rows_of = [&](int j) {
        const int r0 = wrow0 + j * BLOCK_ROWS;
        return (j < RPC && A.k != 0) ? max(0, min(CR, A.n - r0)) : 0;
      };
      auto tissue = [&](int j) {
        const int nr = rows_of(j);
        if (issuer && nr > 0) {
          const unsigned bytes = (unsigned)(nr * GW * sizeof(S));
          const size_t off = (size_t)g * A.ld * GW + (size_t)(wrow0 + j * BLOCK_ROWS) * GW;
          const bool t2 = A.k >= 2, ac = A.acc_terms > 0 && !A.acc_init;
          unsigned long long* bar = &s_bar[bw][j % STG];
          fence_proxy_async();
          mbar_expect_tx(bar, bytes * (1u + (t2 ? 1u : 0u) + (ac ? 1u : 0u)));
          S* d = &s_pre[j % STG][0][bw * WE];
          bulk_g2s(d, static_cast<const S*>(A.Tprev) + off, bytes, bar);
          if (t2) bulk_g2s(d + PS, static_cast<const S*>(A.Tout) + off, bytes, bar);
          if (ac) bulk_g2s(d + 2 * PS, static_cast<const S*>(A.acc) + off, bytes, bar);
        }
      };
#pragma unroll
      for (int j = 0; j < STG - 1; ++j) tissue(j);
#pragma unroll 1
      for (int j = 0; j < RPC; ++j) {
        // every thread is done with the stage tissue() refills
        if constexpr (TMA == 1) __syncwarp(); else __syncthreads();
        tissue(j + STG - 1);
        if (!GS_ROW_PREFETCH && j > 0) cur = row_idx(j);
        const RowIdx<S> nx = next_idx(j);
        if (rows_of(j) > 0) mbar_wait(&s_bar[bw][j % STG], (unsigned)((j / STG) & 1));
        cheb_row<S, GW, MODE>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er,
                              &s_pre[j % STG][0][threadIdx.x * VEC], PS, cur);
        cur = nx;
      }
      if constexpr (MODE != MODE_NONE) block_epilogue<S, GW, MODE>(A, g, tile, warp, sub, q, mn, mx, er);
      return;
    }
#pragma unroll
    for (int j = 0; j < STG - 1; ++j) issue(j);
#pragma unroll 1
    for (int j = 0; j < RPC; ++j) {
      issue(j + STG - 1);
      if (!GS_ROW_PREFETCH && j > 0) cur = row_idx(j);
      const RowIdx<S> nx = next_idx(j);
      cp_async_wait<STG - 1>();
      cheb_row<S, GW, MODE>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er,
                            &s_pre[j % STG][0][threadIdx.x * VEC], PS, cur, GS_PRE_TP != 0);
      cur = nx;
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < RPC; ++j) {
      if (!GS_ROW_PREFETCH && j > 0) cur = row_idx(j);
      const RowIdx<S> nx = next_idx(j);
      cheb_row<S, GW, MODE>(A, g, base + j * BLOCK_ROWS, sub, q, mn, mx, er, nullptr, 0, cur);
      cur = nx;
    }
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<S, GW, MODE>(A, g, tile, warp, sub, q, mn, mx, er);
}

// One row per lane (B <= 2 fp64, B <= 4 in the 32-bit mode; config 3's one-column Sinkhorn) with the
// CSR stream staged through shared memory. The (col, val) entries of a warp's 32 consecutive rows
// are one contiguous run of both arrays, so lane 0 brings the warp's slice in with two bulk copies
// (cp.async.bulk, completion on the warp's mbarrier): the matrix stream -- 85% of this layout's
// bytes -- is in flight without holding registers, and the lanes' dependent chain shrinks to
// shared-memory index -> gather -> fma. Warps run independently (no CTA barrier in the row loop);
// the next slice's bounds, the next rows' CSR ranges and own-row operands are loaded one row block
// ahead. Same CTA geometry, per-row fma chain and epilogue partials as k_cheb_step (bit-identical
// results); a warp whose slice exceeds its stage (GS_LANE_CAP entries) folds it from global
// memory. The arrays may be the odd-stride copy of gs_lane.cu. sparse.cpp:85-99 / heat.cpp:121-130.
#ifndef GS_LANE_CAP
#define GS_LANE_CAP 736  // entries per warp stage: 23 per row
#endif
#ifndef GS_LANE_MIN_BLOCKS
#define GS_LANE_MIN_BLOCKS 4
#endif
#ifndef GS_LANE_BATCH
#define GS_LANE_BATCH 8  // gathers in flight per lane
#endif
constexpr int kLaneStride = GS_LANE_CAP;  // stage stride (a 16-byte multiple in both arrays)
static_assert(GS_LANE_CAP % 4 == 0, "16-byte stage stride");
template <typename S>
constexpr int lane_smem_bytes() {
  return (kStepThreads / 32) * kLaneStride * (int)(sizeof(int) + sizeof(S));
}

// NB consecutive staged entries of one row folded into its chain (CSR order). TAIL: positions at
// or past `pe` read the row's last index (a valid position) and skip their gather and fma.
template <typename S, int GW, int NB, bool TAIL>
__device__ __forceinline__ void lane_batch(const int* sc, const S* sv, int p, int pe, const S* __restrict__ Tp,
                                           double (&y)[Lay<GW, S>::VEC]) {
  constexpr int VEC = Lay<GW, S>::VEC;
  using P = Prec<S>;
  int at[NB];
  int cc[NB];
  S vv[NB];
  S xx[NB][VEC];
#pragma unroll
  for (int u = 0; u < NB; ++u) at[u] = TAIL ? min(p + u, pe - 1) : p + u;
#pragma unroll
  for (int u = 0; u < NB; ++u) cc[u] = sc[at[u]];
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    if constexpr (TAIL) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) xx[u][e] = S(0);
      if (p + u < pe) ld_vec<S, VEC>(Tp + (size_t)cc[u] * GW, xx[u]);
    } else {
      ld_vec<S, VEC>(Tp + (size_t)cc[u] * GW, xx[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < NB; ++u) vv[u] = sv[at[u]];
#pragma unroll
  for (int u = 0; u < NB; ++u)
    if (!TAIL || p + u < pe) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(vv[u]), P::dec(xx[u][e]), y[e]);
    }
}

// One row's chain from entries [p, pe) of a slice (shared-memory stage or global arrays):
// GS_LANE_BATCH entries at a time -- indices, the gathers, then the values (read while the gathers
// are in flight) and the fma chain in CSR order. A trailing pad entry of the odd-stride copy
// (column -1, gs_lane.cu) is dropped first.
template <typename S, int GW>
__device__ __forceinline__ void lane_fold(const int* sc, const S* sv, int p, int pe, const S* __restrict__ Tp,
                                          double (&y)[Lay<GW, S>::VEC]) {
  constexpr int NB = GS_LANE_BATCH;
  if (pe > p && sc[pe - 1] < 0) --pe;
  for (; p + NB <= pe; p += NB) lane_batch<S, GW, NB, false>(sc, sv, p, pe, Tp, y);
  // the row's tail, predicated
  if (p + NB / 2 < pe) lane_batch<S, GW, NB, true>(sc, sv, p, pe, Tp, y);
  else if (p < pe) lane_batch<S, GW, NB / 2, true>(sc, sv, p, pe, Tp, y);
}

template <typename S, int GW, int MODE>
__global__ void __launch_bounds__(kStepThreads, sizeof(S) == 8 ? 3 : GS_LANE_MIN_BLOCKS) k_cheb_lane(const StepArgs A) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC;
  static_assert(L::LPR == 1, "one row per lane");
  constexpr int RPC = kRowsPerCta1, BLOCK_ROWS = kStepThreads, NW = kStepThreads / 32;
  if (A.status && (A.status->error || A.status->done)) return;
  const int tl = tile_of(A, blockIdx.x / A.Gl);
  const int tile = A.tile0 + tl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ __align__(128) unsigned char lane_smem[];
  int* sc = reinterpret_cast<int*>(lane_smem) + warp * kLaneStride;
  S* sv = reinterpret_cast<S*>(lane_smem + (size_t)NW * kLaneStride * sizeof(int)) + warp * kLaneStride;
  __shared__ __align__(8) unsigned long long s_bar[NW];
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = MODE == MODE_BARY_PSI ? -INFINITY : 0.0;
    er[e] = 0.0;
  }
  const int wbase = A.row0 + tl * (BLOCK_ROWS * RPC) + warp * 32;  // the warp's rows of block 0
  const S* __restrict__ vals = static_cast<const S*>(A.vals);
  const size_t gbase = (size_t)g * A.ld * GW;
  const S* __restrict__ Tp = static_cast<const S*>(A.Tprev) + gbase;
  // the warp's slice of block j: first entry rounded down and length rounded up to four entries
  // (16-byte copies; the arrays carry kCsrPad). len 0 = no rows; > GS_LANE_CAP = not staged
  // (kept as the two loaded offsets, so the loads stay in flight until the bounds are needed)
  struct Slice {
    int a, b;
    __device__ __forceinline__ int p0() const { return a & ~3; }
    __device__ __forceinline__ int len() const { return ((b + 3) & ~3) - (a & ~3); }
  };
  auto slice = [&](int j) {
    Slice sl{0, 0};
    const int r0 = wbase + j * BLOCK_ROWS;
    if (j < RPC && r0 < A.n) {
      sl.a = __ldg(A.offs + r0);
      sl.b = __ldg(A.offs + min(r0 + 32, A.n));
    }
    return sl;
  };
  // a row's CSR range and own-row operands T_{k-1}[i], T_{k-2}[i], acc[i]
  struct RowPre {
    int p, pe;
    S tps[VEC], t2s[VEC], a0s[VEC];
  };
  auto preload = [&](int j) {
    RowPre r;
    r.p = r.pe = 0;
#pragma unroll
    for (int e = 0; e < VEC; ++e) r.tps[e] = r.t2s[e] = r.a0s[e] = S(0);
    const int row = wbase + j * BLOCK_ROWS + lane;
    if (j < RPC && row < A.n) {
      r.p = __ldg(A.offs + row);
      r.pe = __ldg(A.offs + row + 1);
      if (A.k != 0) {
        const size_t idx = gbase + (size_t)row * GW;
        ld_vec<S, VEC>(static_cast<const S*>(A.Tprev) + idx, r.tps);
        if (A.k >= 2) ld_vec_rw<S, VEC>(static_cast<const S*>(A.Tout) + idx, r.t2s);
        if (A.acc_terms > 0 && !A.acc_init) ld_vec_rw<S, VEC>(static_cast<const S*>(A.acc) + idx, r.a0s);
      }
    }
    return r;
  };
  auto issue = [&](const Slice& sl) {  // lane 0: the slice into the warp's stage
    if (lane != 0) return;
    const int p0 = sl.p0(), len = sl.len();
    if (len <= 0 || len > GS_LANE_CAP) return;
    fence_proxy_async();  // the lanes' reads of the stage (ordered by __syncwarp) before the copy's writes
    mbar_expect_tx(&s_bar[warp], (unsigned)(len * (sizeof(int) + sizeof(S))));
    bulk_g2s(sc, A.cols + p0, (unsigned)(len * sizeof(int)), &s_bar[warp]);
    bulk_g2s(sv, vals + p0, (unsigned)(len * sizeof(S)), &s_bar[warp]);
  };
  if (lane == 0) {
    mbar_init(&s_bar[warp], 1);
    fence_proxy_async();
  }
  __syncwarp();
  Slice cs = slice(0);
  issue(cs);
  RowPre cur = preload(0);
  unsigned phase = 0;  // parity of the stage's next completion (oversize slices skip theirs)
#pragma unroll 1
  for (int j = 0; j < RPC; ++j) {
    const int p0 = cs.p0(), len = cs.len();
    if (len <= 0) break;  // past the last row (warp-uniform)
    const int row = wbase + j * BLOCK_ROWS + lane;
    // next block: slice bounds, CSR ranges and own rows in flight during this block's gathers
    const Slice ns = slice(j + 1);
    const RowPre nxt = preload(j + 1);
    const bool valid = row < A.n;
    double y[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) y[e] = 0.0;
    if (len > GS_LANE_CAP) {  // oversize slice (warp-uniform): the same fold from global memory
      if (valid) lane_fold<S, GW>(A.cols + p0, vals + p0, cur.p - p0, cur.pe - p0, Tp, y);
    } else {
      mbar_wait(&s_bar[warp], phase);
      phase ^= 1u;
      if (valid) lane_fold<S, GW>(sc, sv, cur.p - p0, cur.pe - p0, Tp, y);
      __syncwarp();  // every lane is done with the stage before it is refilled
    }
    issue(ns);
    if (valid) {
      if (A.k == 0) st_enc<S, VEC>(static_cast<S*>(A.Tout) + gbase + (size_t)row * GW, y);  // plain SpMM
      else finish_row_ops<S, GW, MODE>(A, g, row, 0, y, mn, mx, er, cur.tps, cur.t2s, cur.a0s);
    }
    cur = nxt;
    cs = ns;
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<S, GW, MODE>(A, g, tile, warp, lane, 0, mn, mx, er);
}

// Several lanes per row, fp64 (B = 3..32 columns: the barycenter layouts of configs 2 and 4) with the
// CSR stream staged through shared memory as 16-byte records {col, -, val} (gs_lane.cu builds the
// record copy). A warp's RPW consecutive rows own one contiguous run of records; lane 0 brings it
// in with one bulk copy (completion on the warp's mbarrier) and every lane reads its row's next
// record with one 16-byte shared-memory load -- a broadcast inside the row's lanes, one wavefront
// per warp -- instead of a coalesced (col, val) chunk load plus three shuffles per entry
// (tools/mb_gather.cu: 240 -> 202 us on a synthetic graph with config 2's shape). On the real kNN
// graphs it wins only for 128-byte rows on the wide-window layout (config 4: 1325 -> 1276 us) and
// is the default there; elsewhere k_cheb_step stays (GS_REC=1 / 0 force). Warps run independently; the
// next slice's bounds and the next rows' own operands are loaded one row block ahead. Same CTA
// geometry, per-row fma chain and epilogue partials as k_cheb_step (bit-identical results); a warp
// whose slice exceeds its stage (GS_REC_CAP records: hub rows) folds it from global memory.
// sparse.cpp:85-99 / heat.cpp:121-130.
#ifndef GS_REC_CAP
#define GS_REC_CAP 256  // records per warp stage (4 KB): config 4 1276 (192) / 1255 (256) / 1466 (384) us
#endif
#ifndef GS_REC_BATCH
#define GS_REC_BATCH 4  // gathers in flight per lane
#endif
#ifndef GS_REC_MIN_BLOCKS
#define GS_REC_MIN_BLOCKS 5
#endif
struct __align__(16) CsrRec {
  int col, pad;
  double val;
};
constexpr int rec_smem_bytes() { return (kStepThreads / 32) * GS_REC_CAP * (int)sizeof(CsrRec); }

// NB consecutive records of one row folded into its chain (CSR order). TAIL: positions at or past
// `pe` read the row's last record instead and skip their fma.
template <typename S, int GW, int NB, bool TAIL>
__device__ __forceinline__ void rec_batch(const CsrRec* sr, int p, int pe, const S* __restrict__ Tp,
                                          double (&y)[Lay<GW, S>::VEC]) {
  constexpr int VEC = Lay<GW, S>::VEC;
  using P = Prec<S>;
  double vv[NB];
  S xx[NB][VEC];
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int4 r = *reinterpret_cast<const int4*>(sr + (TAIL ? min(p + u, pe - 1) : p + u));
    vv[u] = __hiloint2double(r.w, r.z);
    ld_vec<S, VEC>(Tp + (size_t)r.x * GW, xx[u]);
  }
#pragma unroll
  for (int u = 0; u < NB; ++u)
    if (!TAIL || p + u < pe) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) y[e] = P::fmat(vv[u], P::dec(xx[u][e]), y[e]);
    }
}
template <typename S, int GW>
__device__ __forceinline__ void rec_fold(const CsrRec* sr, int p, int pe, const S* __restrict__ Tp,
                                         double (&y)[Lay<GW, S>::VEC]) {
  constexpr int NB = GS_REC_BATCH;
  for (; p + NB <= pe; p += NB) rec_batch<S, GW, NB, false>(sr, p, pe, Tp, y);
  if (p < pe) rec_batch<S, GW, NB, true>(sr, p, pe, Tp, y);
}

template <typename S, int GW, int MODE, int RPC>
__global__ void __launch_bounds__(kStepThreads, Lay<GW, S>::VEC >= 2 ? 4 : GS_REC_MIN_BLOCKS) k_cheb_rec(const StepArgs A) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC, LPR = L::LPR, RPW = L::RPW;
  static_assert(sizeof(S) == 8 && LPR > 1, "fp64 rows shared by several lanes");
  constexpr int BLOCK_ROWS = (kStepThreads / 32) * RPW;
  if (A.status && (A.status->error || A.status->done)) return;
  const int tl = tile_of(A, blockIdx.x / A.Gl);
  const int tile = A.tile0 + tl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  extern __shared__ __align__(128) unsigned char rec_smem[];
  CsrRec* sr = reinterpret_cast<CsrRec*>(rec_smem) + warp * GS_REC_CAP;
  __shared__ __align__(8) unsigned long long s_bar[kStepThreads / 32];
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = MODE == MODE_BARY_PSI ? -INFINITY : 0.0;
    er[e] = 0.0;
  }
  const int wbase = A.row0 + tl * (BLOCK_ROWS * RPC) + warp * RPW;  // the warp's rows of block 0
  const CsrRec* __restrict__ recs = static_cast<const CsrRec*>(A.recs);
  const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
  const S* __restrict__ Tp = static_cast<const S*>(A.Tprev) + gbase;
  struct Slice {  // the warp's records of block j: [a, b)
    int a, b;
  };
  auto slice = [&](int j) {
    Slice sl{0, 0};
    const int r0 = wbase + j * BLOCK_ROWS;
    if (j < RPC && r0 < A.n) {
      sl.a = __ldg(A.offs + r0);
      sl.b = __ldg(A.offs + min(r0 + RPW, A.n));
    }
    return sl;
  };
  struct RowPre {  // a row's record range and own-row operands T_{k-1}[i], T_{k-2}[i], acc[i]
    int p, pe;
    S tps[VEC], t2s[VEC], a0s[VEC];
  };
  auto preload = [&](int j) {
    RowPre r;
    r.p = r.pe = 0;
#pragma unroll
    for (int e = 0; e < VEC; ++e) r.tps[e] = r.t2s[e] = r.a0s[e] = S(0);
    const int row = wbase + j * BLOCK_ROWS + sub;
    if (j < RPC && row < A.n) {
      r.p = __ldg(A.offs + row);
      r.pe = __ldg(A.offs + row + 1);
      if (A.k != 0) {
        const size_t idx = gbase + (size_t)row * GW;
        ld_vec<S, VEC>(static_cast<const S*>(A.Tprev) + idx, r.tps);
        if (A.k >= 2) ld_vec_rw<S, VEC>(static_cast<const S*>(A.Tout) + idx, r.t2s);
        if (A.acc_terms > 0 && !A.acc_init) ld_vec_rw<S, VEC>(static_cast<const S*>(A.acc) + idx, r.a0s);
      }
    }
    return r;
  };
  auto issue = [&](const Slice& sl) {  // lane 0: the slice into the warp's stage
    const int len = sl.b - sl.a;
    if (lane != 0 || len <= 0 || len > GS_REC_CAP) return;
    fence_proxy_async();  // the lanes' reads of the stage (ordered by __syncwarp) before the copy's writes
    mbar_expect_tx(&s_bar[warp], (unsigned)(len * sizeof(CsrRec)));
    bulk_g2s(sr, recs + sl.a, (unsigned)(len * sizeof(CsrRec)), &s_bar[warp]);
  };
  if (lane == 0) {
    mbar_init(&s_bar[warp], 1);
    fence_proxy_async();
  }
  __syncwarp();
  Slice cs = slice(0);
  issue(cs);
  RowPre cur = preload(0);
  unsigned phase = 0;  // parity of the stage's next completion (oversize slices skip theirs)
#pragma unroll 1
  for (int j = 0; j < RPC; ++j) {
    const int len = cs.b - cs.a;
    if (len <= 0) break;  // past the last row (warp-uniform)
    const int row = wbase + j * BLOCK_ROWS + sub;
    Slice ns{0, 0};
    RowPre nxt = cur;
    if constexpr (RPC > 1) {  // next block in flight during this block's gathers
      ns = slice(j + 1);
      nxt = preload(j + 1);
    }
    const bool valid = row < A.n;
    double y[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) y[e] = 0.0;
    if (len > GS_REC_CAP) {  // oversize slice (warp-uniform): the same fold from global memory
      if (valid) rec_fold<S, GW>(recs + cs.a, cur.p - cs.a, cur.pe - cs.a, Tp, y);
    } else {
      mbar_wait(&s_bar[warp], phase);
      phase ^= 1u;
      if (valid) rec_fold<S, GW>(sr, cur.p - cs.a, cur.pe - cs.a, Tp, y);
      __syncwarp();  // every lane is done with the stage before it is refilled
    }
    if constexpr (RPC > 1) issue(ns);
    if (valid) {
      if (A.k == 0) st_enc<S, VEC>(static_cast<S*>(A.Tout) + gbase + (size_t)row * GW, y);  // plain SpMM
      else finish_row_ops<S, GW, MODE>(A, g, row, q, y, mn, mx, er, cur.tps, cur.t2s, cur.a0s);
    }
    cur = nxt;
    cs = ns;
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<S, GW, MODE>(A, g, tile, warp, sub, q, mn, mx, er);
}

// 8-row blocks (wide fp64 rows, one warp per block): the gathers of a block's rows are shared.
// The block's entries are stored re-sorted by (ORIGINAL column, row): every row's entries appear
// in its CSR order (from_triplets sorts rows by original column, sparse.cpp:15-53), so each of
// the 8 per-row fma chains is unchanged -- bit-identical -- while a neighbour row referenced by
// several rows of the block is gathered once. A warp holds the 8 rows' y (2 columns per lane),
// reads 32 records per coalesced load, finds the records that start a new column (ballot), gathers
// those rows GB at a time and folds each record into its row's chain. On config 1's Cuthill-McKee
// order a block references 0.47 distinct rows per entry (SURVEY §8(d) gather model: 1 per entry).
#ifndef GS_BLK_GATHER_BATCH
#define GS_BLK_GATHER_BATCH 4
#endif
#ifndef GS_BLK_MIN_BLOCKS
#define GS_BLK_MIN_BLOCKS 3
#endif
// stage the block's T_{k-2} and acc rows (2 x 4 KB per warp) with TMA bulk copies at block start
#ifndef GS_BLK_STAGE
#define GS_BLK_STAGE 1
#endif
constexpr int kBlkRows = 8;
#ifndef GS_BLK_WARPS
#define GS_BLK_WARPS 4
#endif
constexpr int kBlkWarps = GS_BLK_WARPS;  // warps (8-row blocks) per CTA

template <typename S, int VEC>
__device__ __forceinline__ void blk_fold(S (&y)[kBlkRows][VEC], int r, S v, const S (&x)[VEC]) {
  switch (r) {  // warp-uniform: the record is broadcast
#define GS_BLK_CASE(R)                                                          \
  case R:                                                                       \
    _Pragma("unroll") for (int e = 0; e < VEC; ++e) y[R][e] = Prec<S>::fmat(v, x[e], y[R][e]); \
    break;
    GS_BLK_CASE(0)
    GS_BLK_CASE(1)
    GS_BLK_CASE(2)
    GS_BLK_CASE(3)
    GS_BLK_CASE(4)
    GS_BLK_CASE(5)
    GS_BLK_CASE(6)
    default:
      _Pragma("unroll") for (int e = 0; e < VEC; ++e) y[7][e] = Prec<S>::fmat(v, x[e], y[7][e]);
#undef GS_BLK_CASE
  }
}

template <typename S, int MODE>
__global__ void __launch_bounds__(kBlkWarps * 32, MODE != MODE_NONE ? 0 : GS_BLK_MIN_BLOCKS)
    k_cheb_blk(const StepArgs A) {
  constexpr int GW = 64;
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC;
  static_assert(L::LPR == 32, "one warp per 64-column row");
  constexpr int GB = GS_BLK_GATHER_BATCH;
  if (A.status && (A.status->error || A.status->done)) return;
  const int tl = blockIdx.x / A.Gl;
  const int tile = A.tile0 + tl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = MODE == MODE_BARY_PSI ? -INFINITY : 0.0;  // BARY_PSI: max of the fused log-sum
    er[e] = 0.0;
  }
  const int r0 = A.row0 + (tl * kBlkWarps + warp) * kBlkRows;
  constexpr int RE = kBlkRows * GW;  // elements per staged operand
  __shared__ __align__(128) S s_own[GS_BLK_STAGE ? kBlkWarps : 1][2][GS_BLK_STAGE ? RE : 1];
  __shared__ __align__(8) unsigned long long s_obar[kBlkWarps];
  const int nrows = max(0, min(kBlkRows, A.n - r0));
  const bool t2 = A.k >= 2, ac = A.acc_terms > 0 && !A.acc_init;
  const bool staged = GS_BLK_STAGE && nrows > 0 && A.k != 0 && (t2 || ac);
  if constexpr (GS_BLK_STAGE) {
    if (lane == 0) {
      mbar_init(&s_obar[warp], 1);
      fence_proxy_async();
    }
    __syncwarp();
    if (staged && lane == 0) {
      const unsigned bytes = (unsigned)(nrows * GW * sizeof(S));
      const size_t off = (size_t)g * A.ld * GW + (size_t)r0 * GW;
      mbar_expect_tx(&s_obar[warp], bytes * ((t2 ? 1u : 0u) + (ac ? 1u : 0u)));
      if (t2) bulk_g2s(&s_own[warp][0][0], static_cast<const S*>(A.Tout) + off, bytes, &s_obar[warp]);
      if (ac) bulk_g2s(&s_own[warp][1][0], static_cast<const S*>(A.acc) + off, bytes, &s_obar[warp]);
    }
  }
  if (r0 < A.n) {
    S y[kBlkRows][VEC];
#pragma unroll
    for (int r = 0; r < kBlkRows; ++r)
#pragma unroll
      for (int e = 0; e < VEC; ++e) y[r][e] = S(0);
    const S* __restrict__ Tp = static_cast<const S*>(A.Tprev) + (size_t)g * A.ld * GW + lane * VEC;
    const S* __restrict__ rv = static_cast<const S*>(A.rec_val);
    const int pb = __ldg(A.offs + r0), pe = __ldg(A.offs + min(r0 + kBlkRows, A.n));
    S xc[VEC];  // the row of the column that is current at a chunk boundary
#pragma unroll
    for (int e = 0; e < VEC; ++e) xc[e] = S(0);
    int prevc = -1;
    int key = -1;
    S val = S(0);
    if (pb + lane < pe) {
      key = __ldg(A.rec_key + pb + lane);
      val = __ldg(rv + pb + lane);
    }
    for (int p0 = pb; p0 < pe; p0 += 32) {
      const int cnt = min(32, pe - p0);
      int nkey = -1;  // next chunk, in flight while this one is folded
      S nval = S(0);
      if (p0 + 32 + lane < pe) {
        nkey = __ldg(A.rec_key + p0 + 32 + lane);
        nval = __ldg(rv + p0 + 32 + lane);
      }
      const int col = key >> 3;
      int up = __shfl_up_sync(0xffffffffu, col, 1);
      if (lane == 0) up = prevc;
      unsigned m = __ballot_sync(0xffffffffu, lane < cnt && col != up);
      int u = 0;
      const int first = m ? __ffs(m) - 1 : cnt;
      for (; u < first; ++u)  // records of the column carried over from the last chunk
        blk_fold<S, VEC>(y, __shfl_sync(0xffffffffu, key, u) & 7, __shfl_sync(0xffffffffu, val, u), xc);
      while (m) {
        int pos[GB];
        S xx[GB][VEC];
#pragma unroll
        for (int j = 0; j < GB; ++j) {
          pos[j] = m ? __ffs(m) - 1 : cnt;
          m &= m ? m - 1 : 0u;
          if (pos[j] < cnt) {
            const int c = __shfl_sync(0xffffffffu, col, pos[j]);
            ld_vec<S, VEC>(Tp + (size_t)c * GW, xx[j]);
          }
        }
        const int tail = m ? __ffs(m) - 1 : cnt;
#pragma unroll
        for (int j = 0; j < GB; ++j) {
          if (pos[j] < cnt) {
            const int end = j + 1 < GB ? (pos[j + 1] < cnt ? pos[j + 1] : tail) : tail;
            for (u = pos[j]; u < end; ++u)
              blk_fold<S, VEC>(y, __shfl_sync(0xffffffffu, key, u) & 7, __shfl_sync(0xffffffffu, val, u), xx[j]);
#pragma unroll
            for (int e = 0; e < VEC; ++e) xc[e] = xx[j][e];
          }
        }
      }
      prevc = __shfl_sync(0xffffffffu, col, cnt - 1);
      key = nkey;
      val = nval;
    }
    if (staged) mbar_wait(&s_obar[warp], 0u);
#pragma unroll
    for (int r = 0; r < kBlkRows; ++r)
      if (r0 + r < A.n)
        finish_row<S, GW, MODE>(A, g, r0 + r, lane, y[r], mn, mx, er,
                                staged ? &s_own[GS_BLK_STAGE ? warp : 0][0][(GS_BLK_STAGE ? r * GW : 0) + lane * VEC] : nullptr,
                                GS_BLK_STAGE ? RE : 0, false);
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<S, GW, MODE, kBlkWarps * 32>(A, g, tile, warp, 0, lane, mn, mx, er);
}

// Small one-column problems (config 0: n = 2000, B = 1) are latency-bound: with one row per lane a
// row's ~13 dependent entry loads run back to back. Here a warp takes one row: its lanes load
// 32 entries and their T_{k-1} values in one round, then every lane folds the (val, x) pairs in
// CSR order from shuffles -- the same fma chain -- and lane 0 finishes the row.
template <typename S, int MODE>
__global__ void __launch_bounds__(kThreads) k_cheb_step_w1(const StepArgs A) {
  if (A.status && (A.status->error || A.status->done)) return;
  const int tl = blockIdx.x / A.Gl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = A.row0 + tl * (kThreads / 32) + warp;
  double mn[1] = {INFINITY}, mx[1] = {MODE == MODE_BARY_PSI ? -INFINITY : 0.0}, er[1] = {0.0};
  if (row < A.n) {
    const S* __restrict__ Tp = static_cast<const S*>(A.Tprev) + (size_t)g * A.ld;
    const S* __restrict__ vals = static_cast<const S*>(A.vals);
    const int pb = __ldg(A.offs + row), pe = __ldg(A.offs + row + 1);
    double y[1] = {0.0};
    for (int p0 = pb; p0 < pe; p0 += 32) {
      S v = S(0), x = S(0);
      if (p0 + lane < pe) {
        v = __ldg(vals + p0 + lane);
        x = __ldg(Tp + __ldg(A.cols + p0 + lane));
      }
      const int cnt = min(32, pe - p0);
      for (int u = 0; u < cnt; ++u)
        y[0] = Prec<S>::fmat(Prec<S>::val(__shfl_sync(0xffffffffu, v, u)),
                             Prec<S>::dec(__shfl_sync(0xffffffffu, x, u)), y[0]);
    }
    if (lane == 0) finish_row<S, 1, MODE>(A, g, row, 0, y, mn, mx, er, nullptr, 0);
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<S, 1, MODE, kThreads>(A, g, A.tile0 + tl, warp, lane, 0, mn, mx, er);
}

}  // namespace gsk

// gs_sell.cuh -- the sliced Chebyshev step (k_cheb_sell): L_s stored in jagged slices of C rows
// (SELL-C style, no slice-maximum padding), for the layouts where several rows share a warp.
//
// Reference path: one step of HeatFilter::apply (proj/src/heat.cpp:121-130) over
// SparseSymMatrix::multiply (proj/src/sparse.cpp:85-99). Every row keeps its entries in CSR
// order (from_triplets' column order, sparse.cpp:15-53) and folds them with the same fma chain
// from +0, so results are bit-identical to k_cheb_step (gs_step.cuh) and to the oracle.
//
// Why (configs 2/3/4: 64/128-byte fp64 rows on kNN graphs in R^30, one-column 32-bit rows at
// n = 2e7): k_cheb_step's LPR lanes of a row load LPR consecutive (col, val) entries and
// broadcast them with three shuffles per entry -- as many L1tex wavefronts as the neighbour
// gathers themselves -- and one-row-per-lane layouts read each row's CSR run with scattered
// per-lane loads (config 3: the LSU data pipe 80% busy, two thirds of it on those loads).
//
// Store: slice s holds rows [C s, C s + C) of the layout. Its entries are cut into chunks of JV
// consecutive entries per row (a row's last chunk padded with col = -1, val = 0). Chunk index c
// of the slice stores, back to back, the chunk of every row that has one (len > c JV) in row
// order -- "jagged": rows that have ended take no space. A lane finds its row's position in the
// chunk from a warp ballot (rank among the rows still running), so
//   * every lane of a row reads the row's (col, val) chunk itself: one coalesced 16-byte load of
//     JV columns and 16-byte pieces of JV values per warp and chunk, no shuffles;
//   * the warp's loads of one chunk are contiguous (C x JV x 4 bytes of columns);
//   * the padding is at most JV - 1 entries per row, whatever the spread of row lengths.
// C = 32 / LPR rows per warp; JV = 4 (C <= 8), 2 (C = 16) or 1 (C = 32: 128 bytes of columns per
// warp and entry without any padding).
#pragma once

#include "gs_step.cuh"

namespace gsk {

__host__ __device__ constexpr int sell_jv(int C) { return C >= 32 ? 1 : (C >= 16 ? 2 : 4); }

struct SellArgs {
  const long long* soff;  // nslices + 1 entry offsets (multiples of 4)
  const int* cols;        // jagged columns (-1 = padding)
  const void* vals;       // jagged values, S
  int nslices;
  const int* wstart;      // k_cheb_sellw: warp w of a column group takes slices [wstart[w], wstart[w + 1])
};

#ifndef GS_SELL_STAGE
#define GS_SELL_STAGE 4  // entries per pipeline stage (a multiple of every JV)
#endif
#ifndef GS_SELL_MIN_BLOCKS
#define GS_SELL_MIN_BLOCKS 3
#endif
#ifndef GS_SELL_SPW
#define GS_SELL_SPW 2  // slices per warp of the multi-slice instantiation
#endif
constexpr int kSellSpw = GS_SELL_SPW;

// (col, val) of one pipeline stage of a row: ST entries
template <typename S, int ST>
struct SellMeta {
  int c[ST];
  S v[ST];
};

// JV consecutive columns of a chunk (16-, 8- or 4-byte load)
template <int JV>
__device__ __forceinline__ void sell_ld_cols(const int* p, int (&v)[JV]) {
  if constexpr (JV == 4) {
    const int4 t = __ldg(reinterpret_cast<const int4*>(p));
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
  } else if constexpr (JV == 2) {
    const int2 t = __ldg(reinterpret_cast<const int2*>(p));
    v[0] = t.x;
    v[1] = t.y;
  } else {
    static_assert(JV == 1, "chunk width");
    v[0] = __ldg(p);
  }
}

// Loads the stage starting at entry j0 of the slice's rows; `off` is the slice-relative entry
// offset of chunk j0 / JV and is advanced past the stage's chunks. Every lane loads (rows that
// have ended read the chunk after their rank, inside the store or its tail padding); an entry
// is used only when its index is below the row's length, so nothing here selects on a loaded
// value and the loads stay in flight until the stage is folded.
template <typename S, int C, int JV, int ST>
__device__ __forceinline__ void sell_load(const SellArgs& E, long long O, int j0, int len, int maxlen,
                                          unsigned ltmask, int& off, SellMeta<S, ST>& m) {
  constexpr int LPR = 32 / C;
  constexpr int PV = 16 / (int)sizeof(S) < JV ? 16 / (int)sizeof(S) : JV;  // values per piece
  constexpr int NP = JV / PV;
  const S* __restrict__ vals = static_cast<const S*>(E.vals);
#pragma unroll
  for (int u = 0; u < ST / JV; ++u) {
    const int jc = j0 + u * JV;
    if (jc < maxlen) {  // warp-uniform
      const unsigned bal = __ballot_sync(0xffffffffu, jc < len);
      const int rank = __popc(bal & ltmask) / LPR;
      const int cnt = __popc(bal) / LPR;
      const long long base = O + off;
      int ct[JV];
      sell_ld_cols<JV>(E.cols + base + rank * JV, ct);
#pragma unroll
      for (int e = 0; e < JV; ++e) m.c[u * JV + e] = ct[e];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        S vt[PV];
        ld_vec<S, PV>(vals + base + (long long)p * cnt * PV + rank * PV, vt);
#pragma unroll
        for (int e = 0; e < PV; ++e) m.v[u * JV + p * PV + e] = vt[e];
      }
      off += cnt * JV;
    }
  }
}

// Gathers the stage's neighbour rows (entries past the row's end read the row itself).
template <typename S, int GW, int ST>
__device__ __forceinline__ void sell_gather(const S* __restrict__ Tp, const SellMeta<S, ST>& m, int j0, int len,
                                            int maxlen, int self, S (&x)[ST][Lay<GW, S>::VEC]) {
  constexpr int VEC = Lay<GW, S>::VEC;
#pragma unroll
  for (int u = 0; u < ST; ++u) {
    if (j0 + u < maxlen) {  // warp-uniform
      const int c = j0 + u < len ? m.c[u] : self;
      ld_vec<S, VEC>(Tp + (size_t)c * GW, x[u]);
    }
  }
}

template <typename S, int GW, int ST>
__device__ __forceinline__ void sell_fold(const SellMeta<S, ST>& m, const S (&x)[ST][Lay<GW, S>::VEC], int j0,
                                          int len, double (&y)[Lay<GW, S>::VEC]) {
  constexpr int VEC = Lay<GW, S>::VEC;
  using P = Prec<S>;
#pragma unroll
  for (int u = 0; u < ST; ++u) {
    if (j0 + u < len) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(m.v[u]), P::dec(x[u][e]), y[e]);
    }
  }
}

// One slice (C rows, one per LPR lanes) of one Chebyshev step.
template <typename S, int GW, int MODE>
__device__ __forceinline__ void sell_slice(const StepArgs& A, const SellArgs& E, int g, int s, int sub, int q,
                                           double (&mn)[Lay<GW, S>::VEC], double (&mx)[Lay<GW, S>::VEC],
                                           double (&er)[Lay<GW, S>::VEC]) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC, C = L::RPW, JV = sell_jv(C), ST = GS_SELL_STAGE;
  static_assert(ST % JV == 0, "a stage is whole chunks");
  const int lane = threadIdx.x & 31;
  const unsigned ltmask = (1u << lane) - 1u;
  const int row = s * C + sub;
  const bool valid = row < A.n;
  const long long O = __ldg(E.soff + s);
  int len = 0;
  if (valid) len = __ldg(A.offs + row + 1) - __ldg(A.offs + row);
  const int maxlen = __reduce_max_sync(0xffffffffu, len);
  const int self = valid ? row : 0;
  const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
  const size_t idx = gbase + (size_t)self * GW;
  const S* __restrict__ Tp = static_cast<const S*>(A.Tprev) + gbase;
  // own-row operands first: their DRAM latency overlaps the gathers
  S tps[VEC], t2s[VEC], a0s[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) tps[e] = t2s[e] = a0s[e] = S(0);
  if (valid && A.k != 0) {
    ld_vec<S, VEC>(static_cast<const S*>(A.Tprev) + idx, tps);
    if (A.k >= 2) ld_vec_rw<S, VEC>(static_cast<const S*>(A.Tout) + idx, t2s);
    if (A.acc_terms > 0 && !A.acc_init) ld_vec_rw<S, VEC>(static_cast<const S*>(A.acc) + idx, a0s);
  }
  double y[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) y[e] = 0.0;
  // pipeline: (col, val) two stages ahead, neighbour rows one stage ahead of the fma chain.
  // Three (col, val) buffers and two row buffers rotate by name (no register copies of loaded
  // values, which would wait for the loads): six stages per loop body.
  int off = 0;
  SellMeta<S, ST> m0 = {}, m1 = {}, m2 = {};
  S x0[ST][VEC] = {}, x1[ST][VEC] = {};
  sell_load<S, C, JV, ST>(E, O, 0, len, maxlen, ltmask, off, m0);
  sell_load<S, C, JV, ST>(E, O, ST, len, maxlen, ltmask, off, m1);
  sell_gather<S, GW, ST>(Tp, m0, 0, len, maxlen, self, x0);
  int j0 = 0;
#define GS_SELL_STEP(MA, MB, MC, XA, XB)                                              \
  sell_load<S, C, JV, ST>(E, O, j0 + 2 * ST, len, maxlen, ltmask, off, MC);           \
  sell_gather<S, GW, ST>(Tp, MB, j0 + ST, len, maxlen, self, XB);                     \
  sell_fold<S, GW, ST>(MA, XA, j0, len, y);                                           \
  j0 += ST;                                                                           \
  if (j0 >= maxlen) break;
  while (j0 < maxlen) {
    GS_SELL_STEP(m0, m1, m2, x0, x1)
    GS_SELL_STEP(m1, m2, m0, x1, x0)
    GS_SELL_STEP(m2, m0, m1, x0, x1)
    GS_SELL_STEP(m0, m1, m2, x1, x0)
    GS_SELL_STEP(m1, m2, m0, x0, x1)
    GS_SELL_STEP(m2, m0, m1, x1, x0)
  }
#undef GS_SELL_STEP
  if (!valid) return;
  if (A.k == 0) {  // plain SpMM (sparse.cpp:85-99)
    st_enc<S, VEC>(static_cast<S*>(A.Tout) + idx, y);
    return;
  }
  finish_row_ops<S, GW, MODE>(A, g, row, q, y, mn, mx, er, tps, t2s, a0s);
}

// A CTA covers SPW x 8 consecutive slices of one column group: warp w takes slices
// (tile SPW + j) 8 + w, j < SPW.
template <typename S, int GW, int MODE, int SPW>
__global__ void __launch_bounds__(kStepThreads, MODE != MODE_NONE ? 0 : GS_SELL_MIN_BLOCKS)
    k_cheb_sell(const StepArgs A, const SellArgs E) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC, LPR = L::LPR;
  constexpr int WARPS = kStepThreads / 32;
  if (A.status && (A.status->error || A.status->done)) return;
  const int tl = blockIdx.x / A.Gl;
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
#pragma unroll 1
  for (int j = 0; j < SPW; ++j) {
    const int s = (tl * SPW + j) * WARPS + warp;
    if (s < E.nslices) sell_slice<S, GW, MODE>(A, E, g, s, sub, q, mn, mx, er);
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<S, GW, MODE>(A, g, tile, warp, sub, q, mn, mx, er);
}

// ---- warp-staged variant (rows of at least four lanes: C <= 8, JV = 4) -------------------------
// k_cheb_sell keeps (col, val) stages and gathered rows in registers; at 80 registers only 24
// warps are resident and the index -> gather -> fma chain of a slice (6-7 stages) spends a third
// of its time filling and draining (ncu r02s_sell_c2: 30% warps active, long-scoreboard stall 10.6
// cycles per issue, L1tex 37% busy). Here
//   * a persistent grid: warp w of the grid takes a contiguous run of slices, the runs cut at
//     equal cost (chunks of the longest row + a constant per slice; gs_sell::cpre) so that the
//     degree-sorted windows' long slices do not pile up on a few warps; the assignment is
//     static, so the per-tile error partials are summed in the same order on every run;
//   * lane 0 copies the whole jagged range of the warp's NEXT slice (columns and values are each
//     one contiguous run) into a per-warp shared-memory buffer with two bulk copies on an
//     mbarrier while the current slice runs (double buffer); slices longer than the buffer are
//     staged synchronously in ranges of whole chunks;
//   * (col, val) then come from broadcast LDS.128 right where they are used, so the only
//     long-latency loads are the neighbour-row gathers, kept in a register ring of 4 DC entries
//     per lane: entry j is folded and entry j + 4 DC is issued into the same registers.
#ifndef GS_SELLW_CAP
#define GS_SELLW_CAP 192  // entries per staged range
#endif
#ifndef GS_SELLW_MIN_BLOCKS
#define GS_SELLW_MIN_BLOCKS 4
#endif
constexpr int kSellwCap = GS_SELLW_CAP;
static_assert(kSellwCap % 4 == 0 && kSellwCap >= 32, "staging buffer: whole chunks of every row");

template <typename S>
struct SellwBuf {  // one staging buffer: columns, values (16 bytes of slack after each)
  static constexpr int COL_BYTES = kSellwCap * 4 + 16;
  static constexpr int VAL_BYTES = kSellwCap * (int)sizeof(S) + 16;
  static constexpr int BYTES = COL_BYTES + VAL_BYTES;
};

// Chunks [c0, c1) of the lane's row from the staged range (sc, sv: its columns / values).
template <typename S, int GW, int DC>
__device__ __forceinline__ void sellw_range(const int* sc, const S* sv, int c0, int c1, int len, int self,
                                            const S* __restrict__ Tp, unsigned ltmask,
                                            double (&y)[Lay<GW, S>::VEC]) {
  using L = Lay<GW, S>;
  using P = Prec<S>;
  constexpr int VEC = L::VEC, LPR = L::LPR;
  constexpr int PV = 16 / (int)sizeof(S) < 4 ? 16 / (int)sizeof(S) : 4, NP = 4 / PV;
  S x[4 * DC][VEC];
  int off_g = 0, off_f = 0;
#pragma unroll
  for (int d = 0; d < DC; ++d) {  // ring fill: chunks c0 .. c0 + DC - 1
    const int c = c0 + d;
    if (c < c1) {
      const unsigned bal = __ballot_sync(0xffffffffu, 4 * c < len);
      const int rank = __popc(bal & ltmask) / LPR, cnt = __popc(bal) / LPR;
      const int4 cc = *reinterpret_cast<const int4*>(sc + off_g + rank * 4);
      off_g += cnt * 4;
      const int ci[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) ld_vec<S, VEC>(Tp + (size_t)(4 * c + u < len ? ci[u] : self) * GW, x[4 * d + u]);
    }
  }
  for (int c = c0; c < c1; c += DC) {
#pragma unroll
    for (int d = 0; d < DC; ++d) {
      const int cf = c + d;  // chunk folded now; chunk cf + DC is gathered into its registers
      if (cf < c1) {         // warp-uniform
        const unsigned balf = __ballot_sync(0xffffffffu, 4 * cf < len);
        const int rankf = __popc(balf & ltmask) / LPR, cntf = __popc(balf) / LPR;
        S v[4];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          S vt[PV];
          ld_vec_rw<S, PV>(sv + off_f + p * cntf * PV + rankf * PV, vt);
#pragma unroll
          for (int e = 0; e < PV; ++e) v[p * PV + e] = vt[e];
        }
        off_f += cntf * 4;
        const int cg = cf + DC;
        const bool have = cg < c1;  // warp-uniform
        int ci[4] = {0, 0, 0, 0};
        if (have) {
          const unsigned balg = __ballot_sync(0xffffffffu, 4 * cg < len);
          const int rankg = __popc(balg & ltmask) / LPR, cntg = __popc(balg) / LPR;
          const int4 cc = *reinterpret_cast<const int4*>(sc + off_g + rankg * 4);
          off_g += cntg * 4;
          ci[0] = cc.x;
          ci[1] = cc.y;
          ci[2] = cc.z;
          ci[3] = cc.w;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (4 * cf + u < len) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(v[u]), P::dec(x[4 * d + u][e]), y[e]);
          }
          if (have) ld_vec<S, VEC>(Tp + (size_t)(4 * cg + u < len ? ci[u] : self) * GW, x[4 * d + u]);
        }
      }
    }
  }
}

template <typename S, int GW, int MODE>
__global__ void __launch_bounds__(kStepThreads, MODE != MODE_NONE ? 0 : GS_SELLW_MIN_BLOCKS)
    k_cheb_sellw(const StepArgs A, const SellArgs E) {
  using L = Lay<GW, S>;
  constexpr int VEC = L::VEC, LPR = L::LPR, C = L::RPW;
  static_assert(sell_jv(C) == 4, "warp-staged slices use chunks of four entries");
  constexpr int WARPS = kStepThreads / 32;
  constexpr int DC = VEC * (int)sizeof(S) >= 16 ? 1 : 2;  // 16-byte lanes: ring of 4; 8-byte: 8
  using B = SellwBuf<S>;
  __shared__ __align__(128) unsigned char s_buf[WARPS][2][B::BYTES];
  __shared__ __align__(8) unsigned long long s_bar[WARPS][2];
  if (A.status && (A.status->error || A.status->done)) return;
  const int tl = blockIdx.x / A.Gl;
  const int tile = A.tile0 + tl;
  const int g = A.g0 + blockIdx.x % A.Gl;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  const unsigned ltmask = (1u << lane) - 1u;
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = MODE == MODE_BARY_PSI ? -INFINITY : 0.0;  // BARY_PSI: max of the fused log-sum
    er[e] = 0.0;
  }
  if (lane == 0) {
    mbar_init(&s_bar[warp][0], 1);
    mbar_init(&s_bar[warp][1], 1);
    fence_proxy_async();
  }
  __syncwarp();
  const S* __restrict__ gvals = static_cast<const S*>(E.vals);
  unsigned ph0 = 0, ph1 = 0;                       // phase parity of the two buffers
  auto stage = [&](int b, long long O, int cnt) {  // bulk copies of `cnt` entries from entry O
    if (lane == 0) {
      unsigned char* d = s_buf[warp][b];
      mbar_expect_tx(&s_bar[warp][b], (unsigned)cnt * (4u + (unsigned)sizeof(S)));
      bulk_g2s(d, E.cols + O, (unsigned)cnt * 4u, &s_bar[warp][b]);
      bulk_g2s(d + B::COL_BYTES, gvals + O, (unsigned)cnt * (unsigned)sizeof(S), &s_bar[warp][b]);
    }
  };
  auto wait = [&](int b) {
    if (b == 0) {
      mbar_wait(&s_bar[warp][0], ph0);
      ph0 ^= 1u;
    } else {
      mbar_wait(&s_bar[warp][1], ph1);
      ph1 ^= 1u;
    }
  };
  int s = __ldg(E.wstart + tl * WARPS + warp);
  const int send = __ldg(E.wstart + tl * WARPS + warp + 1);
  long long O = 0;
  int sz = 0;
  if (s < send) {
    O = __ldg(E.soff + s);
    sz = (int)min((long long)INT32_MAX, __ldg(E.soff + s + 1) - O);
    if (sz > 0 && sz <= kSellwCap) stage(0, O, sz);
  }
  int b = 0;
#pragma unroll 1
  for (; s < send; ++s, b ^= 1) {
    // next slice: its range is copied into the other buffer while this one runs
    const int sn = s + 1;
    long long On = 0;
    int szn = 0;
    if (sn < send) {
      On = __ldg(E.soff + sn);
      szn = (int)min((long long)INT32_MAX, __ldg(E.soff + sn + 1) - On);
      if (szn > 0 && szn <= kSellwCap) stage(b ^ 1, On, szn);
    }
    const int row = s * C + sub;
    const bool valid = row < A.n;
    int len = 0;
    if (valid) len = __ldg(A.offs + row + 1) - __ldg(A.offs + row);
    const int maxlen = __reduce_max_sync(0xffffffffu, len);
    const int nch = (maxlen + 3) >> 2;
    const int self = valid ? row : 0;
    const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
    const size_t idx = gbase + (size_t)self * GW;
    const S* __restrict__ Tp = static_cast<const S*>(A.Tprev) + gbase;
    S tps[VEC], t2s[VEC], a0s[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) tps[e] = t2s[e] = a0s[e] = S(0);
    if (valid && A.k != 0) {  // own-row operands: in flight under the gathers
      ld_vec<S, VEC>(static_cast<const S*>(A.Tprev) + idx, tps);
      if (A.k >= 2) ld_vec_rw<S, VEC>(static_cast<const S*>(A.Tout) + idx, t2s);
      if (A.acc_terms > 0 && !A.acc_init) ld_vec_rw<S, VEC>(static_cast<const S*>(A.acc) + idx, a0s);
    }
    double y[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) y[e] = 0.0;
    const int* sc = reinterpret_cast<const int*>(s_buf[warp][b]);
    const S* sv = reinterpret_cast<const S*>(s_buf[warp][b] + B::COL_BYTES);
    if (sz > 0 && sz <= kSellwCap) {
      wait(b);
      sellw_range<S, GW, DC>(sc, sv, 0, nch, len, self, Tp, ltmask, y);
    } else if (sz > 0) {  // long slice: ranges of whole chunks, staged one after another
      long long Oc = O;
      for (int c0 = 0; c0 < nch;) {
        int c1 = c0, ne = 0;
        while (c1 < nch) {
          const int cnt = __popc(__ballot_sync(0xffffffffu, 4 * c1 < len)) / LPR * 4;
          if (ne + cnt > kSellwCap) break;
          ne += cnt;
          ++c1;
        }
        __syncwarp();  // the previous range is folded: the buffer may be overwritten
        stage(b, Oc, ne);
        wait(b);
        sellw_range<S, GW, DC>(sc, sv, c0, c1, len, self, Tp, ltmask, y);
        Oc += ne;
        c0 = c1;
      }
    }
    if (valid) {
      if (A.k == 0) st_enc<S, VEC>(static_cast<S*>(A.Tout) + idx, y);  // plain SpMM (sparse.cpp:85-99)
      else finish_row_ops<S, GW, MODE>(A, g, row, q, y, mn, mx, er, tps, t2s, a0s);
    }
    __syncwarp();  // every lane is done with buffer b before it is refilled
    O = On;
    sz = szn;
  }
  if constexpr (MODE != MODE_NONE) block_epilogue<S, GW, MODE>(A, g, tile, warp, sub, q, mn, mx, er);
}

}  // namespace gsk

// gs_win.cuh -- the windowed Chebyshev step (k_cheb_win): neighbour rows of T_{k-1} staged in a
// shared-memory window by TMA gathers, on a precomputed per-CTA schedule (gs_win.cu).
//
// Reference path: one step of HeatFilter::apply (proj/src/heat.cpp:121-130) over
// SparseSymMatrix::multiply (proj/src/sparse.cpp:85-99); same per-row fma chain as k_cheb_step
// (gs_step.cuh), so results are bit-identical to it and to the oracle.
//
// Why: k_cheb_step gathers every neighbour row through L1 (3 shuffles per CSR entry to broadcast
// (col, val), ~45% L1 hit rate) and is bound by the L1tex data pipe and by the latency of the
// dependent index -> gather chain. Here:
//   * one persistent CTA per SM owns a contiguous range of rows of the window layout (a recursive
//     BFS-bisection vertex order, so a range is a compact patch of the graph);
//   * the range is cut into row blocks; for each block the schedule lists the neighbour rows that
//     are not already in the CTA's shared-memory ring of W rows ("loads"), in groups of four;
//   * a producer warp issues one `cp.async.bulk.tensor.2d.tile::gather4` per group (four
//     512-byte rows per instruction into four consecutive ring slots) plus three bulk copies of
//     the block's CSR values, ring-slot indices and row offsets, all on the block's mbarrier,
//     `kWinStages` blocks ahead of the consumers;
//   * consumer warps fold each row's entries in CSR order from the ring (broadcast LDS of the
//     value and slot, LDS.128 of the row slice) -- no shuffles, no global gathers;
//   * the own-row operands T_{k-2}[i] and acc[i] are read from global memory into registers at the
//     start of the row; T_{k-1}[i] comes from the ring (every row's own vertex is scheduled);
//   * ring-slot reuse is decided offline with the producer's lead bounded by kWinStages blocks, so
//     a slot is never overwritten while a block that reads it may still be in flight.
// On config 1 the bisection order brings the loads to ~0.12 per CSR entry (each neighbour row is
// fetched ~1.6 times per step instead of once per entry).
#pragma once

#include <cuda.h>

#include "gs_step.cuh"

namespace gsk {

struct WinBlk {  // one row block of the schedule (32 bytes)
  int row0, nrows;  // rows [row0, row0 + nrows) of the window layout
  int lbeg, nl;     // its loads: loads[lbeg .. lbeg + nl), nl % 4 == 0
  int slot0;        // ring slot of its first load (consecutive slots, modulo W)
  int e0, e1;       // padded CSR entry range of its rows
  int wait;         // the producer issues this block once block `wait` is consumed (< the CTA's
                    // first block: no wait)
};

#ifndef GS_WIN_WARPS
#define GS_WIN_WARPS 16
#endif
#ifndef GS_WIN_STAGES
#define GS_WIN_STAGES 3
#endif
#ifndef GS_WIN_EMAX
#define GS_WIN_EMAX 1024
#endif
#ifndef GS_WIN_LMAX_CAP
#define GS_WIN_LMAX_CAP 1024
#endif
// dynamic shared memory of one CTA (the B200 opt-in maximum is 227 KB = 232448 bytes)
#ifndef GS_WIN_SMEM_BYTES
#define GS_WIN_SMEM_BYTES 232448
#endif
constexpr int kWinWarps = GS_WIN_WARPS;    // consumer warps per CTA (+ one producer warp)
constexpr int kWinStages = GS_WIN_STAGES;  // blocks in flight (producer lead + 1)
constexpr int kWinEmax = GS_WIN_EMAX;      // CSR entries per block at most
constexpr int kWinLmaxCap = GS_WIN_LMAX_CAP;  // loads per block at most (the plan: W / 4)
constexpr int kWinThreads = (kWinWarps + 1) * 32;

__host__ __device__ constexpr int win_align16(int b) { return (b + 15) & ~15; }

// Per-stage metadata area: values, slots, row offsets and own slots of one block. The schedule's
// CSR copy pads every row to a multiple of four entries ("quads"), so a consumer reads four
// values with one or two broadcast LDS.128 and four ring slots with one LDS.64.
constexpr int kWinRowsMax = 256;  // rows per block at most
template <typename S>
struct WinMeta {
  static constexpr int VAL_BYTES = win_align16((kWinEmax + 8) * (int)sizeof(S));
  static constexpr int SLOT_BYTES = win_align16((kWinEmax + 16) * 2);
  static constexpr int ROWS_MAX = kWinRowsMax;
  static constexpr int OFF_BYTES = win_align16((ROWS_MAX + 8) * 4);
  static constexpr int OWN_BYTES = win_align16((ROWS_MAX + 16) * 2);
  static constexpr int BYTES = VAL_BYTES + SLOT_BYTES + OFF_BYTES + OWN_BYTES;
};

// ring slots for a row of `row_bytes` bytes: the shared memory left after the stage metadata and
// the barriers (a multiple of 4, at most 65532)
template <typename S>
__host__ __device__ constexpr int win_ring_slots(int row_bytes) {
  return ((((GS_WIN_SMEM_BYTES - kWinStages * WinMeta<S>::BYTES - 2 * kWinStages * 8) / row_bytes) & ~3) > 65532)
             ? 65532
             : (((GS_WIN_SMEM_BYTES - kWinStages * WinMeta<S>::BYTES - 2 * kWinStages * 8) / row_bytes) & ~3);
}

template <typename S, int GW>
constexpr int win_smem_bytes() {
  return win_ring_slots<S>(GW * (int)sizeof(S)) * GW * (int)sizeof(S) + kWinStages * WinMeta<S>::BYTES +
         2 * kWinStages * 8;
}
static_assert(win_smem_bytes<double, 64>() <= GS_WIN_SMEM_BYTES, "window shared memory");

struct WinArgs {
  const WinBlk* blk;
  const int* cta_blk;            // [nctas + 1]: the CTA's blocks
  const int* loads;              // row ids, groups of four
  // the layout's CSR with every row padded to whole quads: poffs[r] = padded start of row r
  // (a multiple of 4) + the row's number of padding entries (0..3)
  const int* poffs;              // n + 1 (+8 padding for the aligned copies)
  const void* pvals;             // values (S), padding entries 0
  const unsigned short* slot;    // ring slot of every padded entry (+16 padding)
  const unsigned short* own;     // ring slot of every row's own T_{k-1} row (+16 padding)
  int W;                         // ring slots
  int nctas;
  unsigned long long* ctatime;   // diagnostics (GS_WIN_CTATIME): per CTA start / end globaltimer
};

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int c0, int4 r,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w),
      "r"(smem_u32(bar))
      : "memory");
}

template <typename S, int VEC>
__device__ __forceinline__ void lds_vec(const S* p, S (&v)[VEC]) {
  if constexpr (VEC * sizeof(S) == 16) {
    if constexpr (sizeof(S) == 8) {
      const double2 t = *reinterpret_cast<const double2*>(p);
      v[0] = t.x;
      v[1] = t.y;
    } else {
      const float4 t = *reinterpret_cast<const float4*>(p);
      v[0] = t.x;
      v[1] = t.y;
      v[2] = t.z;
      v[3] = t.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) v[e] = p[e];
  }
}

// CTA fold of the epilogue partials (as block_epilogue, on a shared-memory area of
// 3 * NWARPS * GW doubles aliased on the ring once every block is consumed).
template <typename S, int GW, int MODE, int NWARPS>
__device__ __forceinline__ void win_epilogue(const StepArgs& A, int g, int tile, int warp, int sub, int q,
                                             double (&mn)[Lay<GW, S>::VEC], double (&mx)[Lay<GW, S>::VEC],
                                             double (&er)[Lay<GW, S>::VEC], double* sm) {
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
  double* s_mn = sm;
  double* s_mx = sm + NWARPS * GW;
  double* s_er = sm + 2 * NWARPS * GW;
  if (sub == 0) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      s_mn[warp * GW + q * VEC + e] = mn[e];
      s_mx[warp * GW + q * VEC + e] = mx[e];
      s_er[warp * GW + q * VEC + e] = er[e];
    }
  }
  __syncthreads();
  if (threadIdx.x < GW) {
    const int c = threadIdx.x;
    double a_mn = s_mn[c], a_mx = s_mx[c], a_er = s_er[c];
    for (int w = 1; w < NWARPS; ++w) {
      a_mn = fmin(a_mn, s_mn[w * GW + c]);
      a_mx = fmax(a_mx, s_mx[w * GW + c]);
      a_er = a_er + s_er[w * GW + c];
    }
    const int col = g * GW + c;
    atomicMin(A.cs.cmin + col, dkey(a_mn));
    if constexpr (MODE == MODE_SK_PSI || MODE == MODE_SK_PHI) atomicMax(A.cs.cmax + col, dkey(a_mx));
    if constexpr (MODE == MODE_BARY_PSI)
      if (A.lbmax && c == 0) atomicMax(A.lbmax, dkey(a_mx));  // max of the fused log-sum
    if constexpr (MODE == MODE_SK_PHI) A.cs.part_err[(size_t)tile * A.Bpad + col] = a_er;
  }
}

// One Chebyshev step over the window layout. Grid: nctas x column groups; one CTA per SM.
template <typename S, int GW, int MODE>
__global__ void __launch_bounds__(kWinThreads, 1)
    k_cheb_win(const __grid_constant__ CUtensorMap tmap, const StepArgs A, const WinArgs WA) {
  using L = Lay<GW, S>;
  using P = Prec<S>;
  using M = WinMeta<S>;
  constexpr int VEC = L::VEC, LPR = L::LPR, RPW = L::RPW;
  constexpr int ROWB = GW * (int)sizeof(S);
  constexpr int NST = kWinStages;
  static_assert(VEC * (int)sizeof(S) == 16 || VEC * (int)sizeof(S) == 8, "8- or 16-byte lanes");
  if (A.status && (A.status->error || A.status->done)) return;
  const int cta = blockIdx.x % WA.nctas;
  const int g = blockIdx.x / WA.nctas;
  if (A.cs.gactive && A.cs.gactive[g] == 0) return;
  extern __shared__ __align__(128) unsigned char smem[];
  if (WA.ctatime && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    WA.ctatime[2 * blockIdx.x] = t;
  }
  const int W = WA.W;
  S* ring = reinterpret_cast<S*>(smem);
  unsigned char* meta = smem + (size_t)W * ROWB;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(meta + NST * M::BYTES);
  unsigned long long* empty = full + NST;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWinWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int b0 = __ldg(WA.cta_blk + cta), b1 = __ldg(WA.cta_blk + cta + 1);
  double mn[VEC], mx[VEC], er[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    mn[e] = INFINITY;
    mx[e] = MODE == MODE_BARY_PSI ? -INFINITY : 0.0;  // BARY_PSI: max of the fused log-sum
    er[e] = 0.0;
  }
  const int64_t grow = (int64_t)g * A.ld;  // first tensor-map row of this column group
  if (warp == kWinWarps) {
    // ---------------- producer ----------------
    // The block's row ids (groups of four) are loaded one block ahead into registers, so the
    // TMA issue never waits on the index loads (up to 32 x U groups per block).
    constexpr int U = (kWinLmaxCap / 4 + 31) / 32;
    int4 ic[U], inx[U];
    auto load_idx = [&](int j, int4 (&dst)[U]) {
      const int ng = j < b1 ? (WA.blk[j].nl >> 2) : 0;
      const int4* src = j < b1 ? reinterpret_cast<const int4*>(WA.loads + WA.blk[j].lbeg) : nullptr;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = lane + 32 * u;
        dst[u] = i < ng ? __ldg(src + i) : make_int4(0, 0, 0, 0);
      }
    };
    load_idx(b0, ic);
    for (int j = b0; j < b1; ++j) {
      const int jj = j - b0, s = jj % NST;
      load_idx(j + 1, inx);
      const WinBlk bk = WA.blk[j];
      if (bk.wait >= b0) {  // every block up to bk.wait consumed (its empty phase completed)
        const int wj = bk.wait - b0;
        mbar_wait(&empty[wj % NST], (unsigned)((wj / NST) & 1));
      }
      unsigned char* mt = meta + s * M::BYTES;
      // e0, e1: padded entry range (multiples of 4)
      const int sb = bk.e0 & ~7, ob = bk.row0 & ~3, wb = bk.row0 & ~7;
      const unsigned vbytes = (unsigned)((bk.e1 - bk.e0) * (int)sizeof(S));
      const unsigned sbytes = bk.e1 > bk.e0 ? (unsigned)win_align16((bk.e1 - sb) * 2) : 0u;
      const unsigned obytes = (unsigned)win_align16((bk.row0 + bk.nrows + 1 - ob) * 4);
      const unsigned wbytes = (unsigned)win_align16((bk.row0 + bk.nrows - wb) * 2);
      if (lane == 0) {
        mbar_expect_tx(&full[s], (unsigned)bk.nl * ROWB + vbytes + sbytes + obytes + wbytes);
        if (vbytes) bulk_g2s(mt, static_cast<const S*>(WA.pvals) + bk.e0, vbytes, &full[s]);
        if (sbytes) bulk_g2s(mt + M::VAL_BYTES, WA.slot + sb, sbytes, &full[s]);
        bulk_g2s(mt + M::VAL_BYTES + M::SLOT_BYTES, WA.poffs + ob, obytes, &full[s]);
        bulk_g2s(mt + M::VAL_BYTES + M::SLOT_BYTES + M::OFF_BYTES, WA.own + wb, wbytes, &full[s]);
      }
      __syncwarp();
      const int ng = bk.nl >> 2;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = lane + 32 * u;
        if (i < ng) {
          int4 r = ic[u];
          r.x += (int)grow;
          r.y += (int)grow;
          r.z += (int)grow;
          r.w += (int)grow;
          int slot = bk.slot0 + 4 * i;
          if (slot >= W) slot -= W;
          tma_gather4(ring + (size_t)slot * GW, &tmap, 0, r, &full[s]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) ic[u] = inx[u];
    }
  } else {
    // ---------------- consumers ----------------
    // Rows go round-robin over the CTA's (warp, lane group) slots across the whole range, so
    // every slot gets the same number of rows whatever the block sizes; a lane group's next row
    // is known ahead, so its T_{k-2} and acc rows are loaded one row early (DRAM latency hidden
    // behind the current row's fold).
    const size_t gbase = (size_t)g * A.ld * GW + q * VEC;
    constexpr int NSLOT = kWinWarps * RPW;
    const int R0 = b1 > b0 ? WA.blk[b0].row0 : 0;
    const int R1 = b1 > b0 ? WA.blk[b1 - 1].row0 + WA.blk[b1 - 1].nrows : 0;
    const bool read_acc = A.acc_terms > 0 && !A.acc_init;
    const bool read_t2 = A.k >= 2;
    int r = R0 + warp * RPW + sub;
    constexpr bool SK = MODE == MODE_SK_PSI || MODE == MODE_SK_PHI;
    constexpr int NE = SK ? 2 * VEC + 1 : 1;  // epilogue operands: M[row], Vcur[row], a[row]
    S t2s[VEC], a0s[VEC];
    double eps_[NE];
    auto own_ops = [&](int row, S (&t2)[VEC], S (&a0)[VEC], double (&ep)[NE]) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        t2[e] = S(0);
        a0[e] = S(0);
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) ep[e] = 0.0;
      if (row < R1) {
        const size_t idx = gbase + (size_t)row * GW;
        if (read_t2) ld_vec_rw<S, VEC>(static_cast<const S*>(A.Tout) + idx, t2);
        if (read_acc) ld_vec_rw<S, VEC>(static_cast<const S*>(A.acc) + idx, a0);
        if constexpr (SK) {
          double m[VEC];
          ld_vec<double, VEC>(A.M + idx, m);
#pragma unroll
          for (int e = 0; e < VEC; ++e) ep[e] = m[e];
          if constexpr (MODE == MODE_SK_PHI) {
            double v[VEC];
            ld_vec_rw<double, VEC>(A.Vcur + idx, v);
#pragma unroll
            for (int e = 0; e < VEC; ++e) ep[VEC + e] = v[e];
          }
          ep[2 * VEC] = __ldg(A.a + row);
        }
      }
    };
    own_ops(r, t2s, a0s, eps_);
    for (int j = b0; j < b1; ++j) {
      const int jj = j - b0, s = jj % NST;
      const WinBlk bk = WA.blk[j];
      const unsigned char* mt = meta + s * M::BYTES;
      const S* sv = reinterpret_cast<const S*>(mt) - bk.e0;
      const unsigned short* ss = reinterpret_cast<const unsigned short*>(mt + M::VAL_BYTES) - (bk.e0 & ~7);
      const int* so = reinterpret_cast<const int*>(mt + M::VAL_BYTES + M::SLOT_BYTES) - (bk.row0 & ~3);
      const unsigned short* sw =
          reinterpret_cast<const unsigned short*>(mt + M::VAL_BYTES + M::SLOT_BYTES + M::OFF_BYTES) - (bk.row0 & ~7);
      const int rend = bk.row0 + bk.nrows;
      mbar_wait(&full[s], (unsigned)((jj / NST) & 1));
      while (r < rend) {
        const int row = r;
        r += NSLOT;
        S t2n[VEC], a0n[VEC];
        double epn[NE];
        own_ops(r, t2n, a0n, epn);  // next row's operands in flight during this row
        const int pr = so[row], pn = so[row + 1];
        const int qe = pn & ~3, npad = pr & 3;
        const S* rl = ring + q * VEC;
        double y[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) y[e] = 0.0;
        // quads of the padded row: the fma chain runs over the real entries in CSR order; full
        // quads first, then the row's last quad with its 1..3 real entries
        auto quad_meta = [&](int p, S (&vv)[4], int (&sl)[4]) {
          if constexpr (sizeof(S) == 8) {
            const double2 v01 = *reinterpret_cast<const double2*>(sv + p);
            const double2 v23 = *reinterpret_cast<const double2*>(sv + p + 2);
            vv[0] = v01.x;
            vv[1] = v01.y;
            vv[2] = v23.x;
            vv[3] = v23.y;
          } else {
            const float4 v4 = *reinterpret_cast<const float4*>(sv + p);
            vv[0] = v4.x;
            vv[1] = v4.y;
            vv[2] = v4.z;
            vv[3] = v4.w;
          }
          const uint2 s4 = *reinterpret_cast<const uint2*>(ss + p);
          sl[0] = (int)(s4.x & 0xffffu);
          sl[1] = (int)(s4.x >> 16);
          sl[2] = (int)(s4.y & 0xffffu);
          sl[3] = (int)(s4.y >> 16);
        };
        const int pf = npad ? qe - 4 : qe;  // end of the full quads
        int p = pr & ~3;
        for (; p < pf; p += 4) {
          S vv[4];
          int sl[4];
          quad_meta(p, vv, sl);
          S xx[4][VEC];
#pragma unroll
          for (int u = 0; u < 4; ++u) lds_vec<S, VEC>(rl + sl[u] * GW, xx[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(vv[u]), P::dec(xx[u][e]), y[e]);
        }
        if (npad) {
          S vv[4];
          int sl[4];
          quad_meta(p, vv, sl);
          const int cnt = 4 - npad;
          S xx[3][VEC];
#pragma unroll
          for (int u = 0; u < 3; ++u)
            if (u < cnt) lds_vec<S, VEC>(rl + sl[u] * GW, xx[u]);
#pragma unroll
          for (int u = 0; u < 3; ++u)
            if (u < cnt)
#pragma unroll
              for (int e = 0; e < VEC; ++e) y[e] = P::fmat(P::val(vv[u]), P::dec(xx[u][e]), y[e]);
        }
        const size_t idx = gbase + (size_t)row * GW;
        if (A.k == 0) {  // plain SpMM
          st_enc<S, VEC>(static_cast<S*>(A.Tout) + idx, y);
        } else {
          S tps[VEC];
          lds_vec<S, VEC>(rl + (int)sw[row] * GW, tps);
          finish_row_ops<S, GW, MODE>(A, g, row, q, y, mn, mx, er, tps, t2s, a0s, SK ? eps_ : nullptr);
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          t2s[e] = t2n[e];
          a0s[e] = a0n[e];
        }
#pragma unroll
        for (int e = 0; e < NE; ++e) eps_[e] = epn[e];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if constexpr (MODE != MODE_NONE) {
    __syncthreads();  // every block consumed: the ring is free for the fold
    win_epilogue<S, GW, MODE, kWinWarps + 1>(A, g, cta, warp, sub, q, mn, mx, er,
                                              reinterpret_cast<double*>(smem));
  }
  if (WA.ctatime) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      WA.ctatime[2 * blockIdx.x + 1] = t;
    }
  }
}

}  // namespace gsk

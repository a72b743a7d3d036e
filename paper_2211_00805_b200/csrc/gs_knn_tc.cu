// gs_knn_tc.cu -- kNN in R^d (9 <= d <= 31, configs 2 and 4: R^30) with a tcgen05 tensor-core
// pre-filter and an exact fp64 re-rank.
//
// Reference: select_knn (proj/src/graph.cpp:30-71): d2 = max(0, |x_i|^2 + |x_j|^2 - 2 <x_i, x_j>)
// from a Gram GEMM, per-row heap of the k smallest (d2, j), eps_i = |x_i - x_{nb_k}|. The engine's
// exact arithmetic (k_knn in gs_graph.cu, the oracle's formula and order) stays the arbiter: the
// tensor cores only choose a candidate superset, every kept candidate is re-scored in fp64 with
// k_knn's formula and the k smallest (d2, j) are selected, so indices and eps are identical to
// the brute force.
//
// Pre-filter: a'_qj = |x_j|^2 - 2 <x_q, x_j> (the query's own |x_q|^2 does not change its
// ranking) as one bf16 GEMM with fp32 accumulation in TMEM: A rows [x_q, 1], B rows
// [-2 x_j, |x_j|^2], each value split into bf16 hi + lo and the three products hi*hi + hi*lo +
// lo*hi accumulated. Per query |a' - exact| <= D_q = 2^-14 (2 |x_q| max_j |x_j| + max_j |x_j|^2):
// the split residuals and the dropped lo*lo term are <= 2^-15 of |x| |2y| per product, the fp32
// accumulation <= 2^-16 of the summed magnitudes; the largest error measured over the kept
// candidates of 10^6 points in R^30 is 2^-16.8 of the same scale (tools/knn_cal.sh,
// GS_KNN_TC_DEBUG=1). Every CTA owns 128 queries (UMMA M = 128)
// and streams all candidates in tiles of 256 (UMMA N = 256): a producer warp bulk-copies the
// tiles (pre-laid out in the K-major core-matrix order, 4 stages), one thread issues six
// tcgen05.mma per tile into one of two TMEM accumulators, and four epilogue warps (one query row
// per thread, TMEM lanes of their quarter) read the 256 values with tcgen05.ld and keep the 32
// smallest. The 32 kept candidates contain the true k nearest whenever the 32nd kept value
// exceeds the k-th by more than 2 D_q (then every j with exact d2 <= the k-th exact d2 is kept);
// queries that fail the test (dense near-ties) are re-run by the brute force.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gs_internal.cuh"
#include "gs_win.cuh"  // mbarrier / bulk-copy helpers

using namespace gsk;

namespace {

constexpr int TQ = 128;    // queries per CTA (UMMA M)
constexpr int TCN = 256;   // candidates per tile (UMMA N)
constexpr int KP = 32;     // kept candidates per query
constexpr int NSTG = 4;    // candidate-tile stages
constexpr int KD = 32;     // padded feature dimension: d values + the augmented column
constexpr int A_ELEMS = TQ * KD;    // bf16 elements of one A tile (hi or lo): 8 KB
constexpr int B_ELEMS = TCN * KD;   // one B tile: 16 KB
constexpr int kTcThreads = 192;     // warp 0 producer, warp 1 MMA, warps 2-5 epilogue
constexpr size_t kTcSmem = (size_t)2 * A_ELEMS * 2 + (size_t)NSTG * 2 * B_ELEMS * 2 + 256;

// K-major core-matrix layout (no swizzle): 8 rows x 16 bytes per 128-byte core matrix; the four
// K blocks of an 8-row group are consecutive (leading byte offset 128), groups 512 bytes apart
// (stride byte offset); a 256-row tile is two 128-row tiles back to back.
__host__ __device__ __forceinline__ size_t blk_off(int64_t r, int k) {
  return (size_t)(((r >> 3) * 4 + (k >> 3)) * 64 + (r & 7) * 8 + (k & 7));
}

__device__ __forceinline__ void split_bf16(double x, __nv_bfloat16& h, __nv_bfloat16& l) {
  h = __float2bfloat16_rn((float)x);
  l = __float2bfloat16_rn((float)(x - (double)__bfloat162float(h)));
}

__global__ void k_tc_prep(const double* __restrict__ pts, const double* __restrict__ sq, int n, int npad,
                          int d, __nv_bfloat16* Ahi, __nv_bfloat16* Alo, __nv_bfloat16* Bhi,
                          __nv_bfloat16* Blo, unsigned long long* maxkeys /* |x| max, |x|^2 max */) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)npad * KD) return;
  const int64_t r = e / KD;
  const int k = (int)(e % KD);
  const __nv_bfloat16 z = __float2bfloat16_rn(0.0f);
  __nv_bfloat16 ah = z, al = z, bh = z, bl = z;
  if (r < n) {
    if (k < d) {
      const double x = pts[r * d + k];
      split_bf16(x, ah, al);
      split_bf16(-2.0 * x, bh, bl);
    } else if (k == d) {
      ah = __float2bfloat16_rn(1.0f);
      split_bf16(sq[r], bh, bl);
      // |x|^2 >= 0: its bit pattern orders like the value
      atomicMax(&maxkeys[0], (unsigned long long)__double_as_longlong(sqrt(sq[r])));
      atomicMax(&maxkeys[1], (unsigned long long)__double_as_longlong(sq[r]));
    }
  } else if (k == d) {
    bh = __float2bfloat16_rn(1e30f);  // padding candidates: never among the smallest
  }
  const size_t o = blk_off(r, k);
  Ahi[o] = ah;
  Alo[o] = al;
  Bhi[o] = bh;
  Blo[o] = bl;
}

// single-thread roles (producer, MMA issuer) wait with a short sleep between polls, so their
// spinning does not take issue slots from the epilogue warps sharing their SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, unsigned parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}

__device__ __forceinline__ uint64_t umma_desc(const void* p) {
  const uint32_t a = smem_u32(p);
  uint64_t dsc = (uint64_t)((a >> 4) & 0x3FFFu);
  dsc |= (uint64_t)(128u >> 4) << 16;  // leading byte offset: next K core matrix
  dsc |= (uint64_t)(512u >> 4) << 32;  // stride byte offset: next 8-row group
  dsc |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  return dsc;                          // base offset 0, SWIZZLE_NONE
}

// kind::f16, A = B = bf16, D = f32, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TCN >> 3) << 17) |
                            ((uint32_t)(TQ >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, "
      "%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcArgs {
  const __nv_bfloat16* Ahi;
  const __nv_bfloat16* Alo;
  const __nv_bfloat16* Bhi;
  const __nv_bfloat16* Blo;
  int n, ntiles;
  int* cand;    // n x KP kept candidates (ascending a'; -1 = none)
  float* cval;  // their a'
};

__global__ void __launch_bounds__(kTcThreads, 1) k_knn_tc(const TcArgs P) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(sm);                   // hi | lo
  __nv_bfloat16* sB = reinterpret_cast<__nv_bfloat16*>(sm + 2 * A_ELEMS * 2);  // NSTG x (hi | lo)
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + 2 * A_ELEMS * 2 + NSTG * 2 * B_ELEMS * 2);
  unsigned long long* full = bars;
  unsigned long long* empty = bars + NSTG;
  unsigned long long* tfull = bars + 2 * NSTG;
  unsigned long long* tempty = tfull + 2;
  unsigned long long* abar = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(abar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qt = blockIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * 32);
    }
    mbar_init(abar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {  // two 256-column fp32 accumulators = all 512 TMEM columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int T = P.ntiles;
  if (warp == 0) {
    if (lane == 0) {  // ---- producer: the query tile once, candidate tiles through the ring
      mbar_expect_tx(abar, 2 * A_ELEMS * 2);
      bulk_g2s(sA, P.Ahi + (size_t)qt * A_ELEMS, A_ELEMS * 2, abar);
      bulk_g2s(sA + A_ELEMS, P.Alo + (size_t)qt * A_ELEMS, A_ELEMS * 2, abar);
      for (int t = 0; t < T; ++t) {
        const int s = t % NSTG;
        if (t >= NSTG) mbar_wait_sleep(&empty[s], (unsigned)(((t / NSTG) - 1) & 1));
        mbar_expect_tx(&full[s], 2 * B_ELEMS * 2);
        __nv_bfloat16* dst = sB + (size_t)s * 2 * B_ELEMS;
        bulk_g2s(dst, P.Bhi + (size_t)t * B_ELEMS, B_ELEMS * 2, &full[s]);
        bulk_g2s(dst + B_ELEMS, P.Blo + (size_t)t * B_ELEMS, B_ELEMS * 2, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: six tcgen05.mma per tile (hi*hi, hi*lo, lo*hi; K = 2 x 16)
      mbar_wait(abar, 0);
      for (int t = 0; t < T; ++t) {
        const int s = t % NSTG, b = t & 1;
        mbar_wait_sleep(&full[s], (unsigned)((t / NSTG) & 1));
        if (t >= 2) mbar_wait_sleep(&tempty[b], (unsigned)(((t >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * TCN);
        const __nv_bfloat16* bt = sB + (size_t)s * 2 * B_ELEMS;
        uint32_t acc = 0;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const __nv_bfloat16* ap = sA + (p == 2 ? A_ELEMS : 0);
          const __nv_bfloat16* bp = bt + (p == 1 ? B_ELEMS : 0);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            umma_bf16(d, umma_desc(ap + kk * 128), umma_desc(bp + kk * 128), acc);
            acc = 1;
          }
        }
        umma_commit(&empty[s]);
        umma_commit(&tfull[b]);
      }
    }
  } else {
    // ---- epilogue: one query row per thread (its warp's TMEM lane quarter)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int q = qt * TQ + row;
    float bd[KP];
    int bi[KP];
#pragma unroll
    for (int s = 0; s < KP; ++s) {
      bd[s] = INFINITY;
      bi[s] = -1;
    }
    float thr = INFINITY;
    for (int t = 0; t < T; ++t) {
      const int b = t & 1;
      mbar_wait(&tfull[b], (unsigned)((t >> 1) & 1));
      tc_fence_after();
      const int jb = t * TCN;
      for (int c = 0; c < TCN / 32; ++c) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * TCN + c * 32), v);
        // fast path: a 32-bit mask of the values below the current 32nd kept value; the
        // insertion (rare after the first tiles) runs only when some lane of the warp has one
        const int base = jb + c * 32;
        unsigned msk = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) msk |= (v[i] < thr ? 1u : 0u) << i;
        if (q >= base && q < base + 32) msk &= ~(1u << (q - base));  // not the query itself
        if (base + 32 > P.n) msk &= P.n > base ? (0xffffffffu >> (32 - (P.n - base))) : 0u;
        if (__any_sync(0xffffffffu, msk != 0)) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if ((msk >> i) & 1u) {
              const float a = v[i];
              const int j = base + i;
#pragma unroll
              for (int s = KP - 1; s > 0; --s) {
                if (bd[s - 1] > a) {
                  bd[s] = bd[s - 1];
                  bi[s] = bi[s - 1];
                } else if (bd[s] > a) {
                  bd[s] = a;
                  bi[s] = j;
                }
              }
              if (bd[0] > a) {
                bd[0] = a;
                bi[0] = j;
              }
            }
          }
          thr = bd[KP - 1];
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[b]);
    }
    if (q < P.n) {
#pragma unroll
      for (int s = 0; s < KP; ++s) {
        P.cand[(size_t)q * KP + s] = bi[s];
        P.cval[(size_t)q * KP + s] = bd[s];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// exact fp64 re-rank of the kept candidates (k_knn's arithmetic and (d2, j) order); queries whose
// candidate set is not provably a superset go to the brute-force list
template <int KMAX>
__global__ void k_tc_rerank(const double* __restrict__ pts, const double* __restrict__ sq, int n, int d,
                            int k, const int* __restrict__ cand, const float* __restrict__ cval,
                            const unsigned long long* __restrict__ maxkeys, int* __restrict__ nbrs,
                            double* __restrict__ eps, int* __restrict__ fb_list, int* __restrict__ fb_count,
                            unsigned long long* dbg, double dq_scale) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int* cq = cand + (size_t)q * KP;
  const float* vq = cval + (size_t)q * KP;
  // superset test: the 32nd kept value beyond the k-th by more than 2 D_q (or fewer than 32 kept)
  const double xmax = __longlong_as_double((long long)maxkeys[0]);
  const double sqmax = __longlong_as_double((long long)maxkeys[1]);
  const double Dq = dq_scale * (2.0 * sqrt(sq[q]) * xmax + sqmax);
  const bool full = cq[KP - 1] >= 0;
  if (!dbg && full && !((double)vq[KP - 1] > (double)vq[k - 1] + 2.0 * Dq)) {
    fb_list[atomicAdd(fb_count, 1)] = q;
    return;
  }
  const double* xq = pts + (size_t)q * d;
  const double sqq = sq[q];
  double bd[KMAX];
  int bi[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    bd[s] = INFINITY;
    bi[s] = 0x7fffffff;
  }
  for (int c = 0; c < KP; ++c) {
    const int j = cq[c];
    if (j < 0) continue;
    const double* xj = pts + (size_t)j * d;
    double g = 0.0;
    for (int u = 0; u < d; ++u) g = fma(xq[u], xj[u], g);
    double d2 = (sqq + sq[j]) - 2.0 * g;
    if (!(d2 > 0.0)) d2 = 0.0;
    if (dbg) {  // calibration: |a' - exact a'| relative to the magnitudes the error scales with
      const double ex = sq[j] - 2.0 * g;
      const double rel = fabs((double)vq[c] - ex) / (2.0 * sqrt(sqq) * sqrt(sq[j]) + sq[j]);
      atomicMax(dbg, (unsigned long long)__double_as_longlong(rel));
    }
    // keep the k smallest (d2, j) pairs in lexicographic order (= the brute force's ascending
    // candidate scan with strict comparisons); k_knn's predicated insertion
#pragma unroll
    for (int s = KMAX - 1; s > 0; --s) {
      if (s < k) {
        if (d2 < bd[s - 1] || (d2 == bd[s - 1] && j < bi[s - 1])) {
          bd[s] = bd[s - 1];
          bi[s] = bi[s - 1];
        } else if (d2 < bd[s] || (d2 == bd[s] && j < bi[s])) {
          bd[s] = d2;
          bi[s] = j;
        }
      }
    }
    if (d2 < bd[0] || (d2 == bd[0] && j < bi[0])) {
      bd[0] = d2;
      bi[0] = j;
    }
  }
  int last = 0;
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    if (s < k) nbrs[(size_t)q * k + s] = bi[s];
    if (s == k - 1) last = bi[s];
  }
  const double* xl = pts + (size_t)last * d;
  double s2 = 0.0;
  for (int u = 0; u < d; ++u) {
    const double diff = xq[u] - xl[u];
    s2 = fma(diff, diff, s2);
  }
  eps[q] = sqrt(s2);
}

}  // namespace

int gs_knn_tc(gs_ctx* ctx, const double* dpts, const double* sq, int n, int d, int k, int* dnb,
              double* deps) {
  cudaStream_t s = ctx->stream;
  if (d + 1 > KD || k > 24) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "tensor-core kNN: d <= 31, k <= 24");
  const int npad = (n + TCN - 1) / TCN * TCN;
  const int qtiles = (n + TQ - 1) / TQ;
  DevBuf<__nv_bfloat16> Ahi, Alo, Bhi, Blo;
  DevBuf<unsigned long long> maxk;
  DevBuf<int> cand, fb, fbn;
  DevBuf<float> cval;
  const size_t elems = (size_t)npad * KD;
  GS_CUDA(ctx, Ahi.alloc(elems, s));
  GS_CUDA(ctx, Alo.alloc(elems, s));
  GS_CUDA(ctx, Bhi.alloc(elems, s));
  GS_CUDA(ctx, Blo.alloc(elems, s));
  GS_CUDA(ctx, maxk.alloc(2, s));
  GS_CUDA(ctx, cand.alloc((size_t)n * KP, s));
  GS_CUDA(ctx, cval.alloc((size_t)n * KP, s));
  GS_CUDA(ctx, fb.alloc(n, s));
  GS_CUDA(ctx, fbn.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(maxk.get(), 0, 2 * sizeof(unsigned long long), s));
  GS_CUDA(ctx, cudaMemsetAsync(fbn.get(), 0, sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_tc_prep<<<(unsigned)((elems + 255) / 256), 256, 0, s>>>(dpts, sq, n, npad, d, Ahi.get(), Alo.get(), Bhi.get(),
                                                           Blo.get(), maxk.get());
  gs_launch_end(ctx, 1);
  static std::vector<char> seen;  // the attribute is per device
  gs_once_per_device(seen, [] { cudaFuncSetAttribute(k_knn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem); });
  TcArgs P{};
  P.Ahi = Ahi.get();
  P.Alo = Alo.get();
  P.Bhi = Bhi.get();
  P.Blo = Blo.get();
  P.n = n;
  P.ntiles = npad / TCN;
  P.cand = cand.get();
  P.cval = cval.get();
  gs_launch_begin(ctx, 1);
  k_knn_tc<<<qtiles, kTcThreads, kTcSmem, s>>>(P);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaGetLastError());
  // D_q scale (GS_KNN_TC_DQ: a power-of-two exponent); GS_KNN_TC_DEBUG=1 measures the largest
  // relative pre-filter error over the kept candidates instead of testing (calibration only)
  const char* dqe = getenv("GS_KNN_TC_DQ");
  const double dq_scale = std::ldexp(1.0, dqe ? atoi(dqe) : -14);
  const bool dbg_on = getenv("GS_KNN_TC_DEBUG") && atoi(getenv("GS_KNN_TC_DEBUG")) != 0;
  DevBuf<unsigned long long> dbg;
  GS_CUDA(ctx, dbg.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(dbg.get(), 0, sizeof(unsigned long long), s));
  gs_launch_begin(ctx, 1);
  if (k <= 16)
    k_tc_rerank<16><<<(n + 127) / 128, 128, 0, s>>>(dpts, sq, n, d, k, cand.get(), cval.get(), maxk.get(), dnb,
                                                    deps, fb.get(), fbn.get(), dbg_on ? dbg.get() : nullptr,
                                                    dq_scale);
  else
    k_tc_rerank<24><<<(n + 127) / 128, 128, 0, s>>>(dpts, sq, n, d, k, cand.get(), cval.get(), maxk.get(), dnb,
                                                    deps, fb.get(), fbn.get(), dbg_on ? dbg.get() : nullptr,
                                                    dq_scale);
  gs_launch_end(ctx, 1);
  if (dbg_on) {
    unsigned long long h = 0;
    GS_CUDA(ctx, cudaMemcpyAsync(&h, dbg.get(), sizeof h, cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    double rel;
    memcpy(&rel, &h, sizeof rel);
    fprintf(stderr, "[gs_knn_tc] max |a' - exact| / (2|x||y| + |y|^2) over kept candidates: %.3e (2^%.2f)\n", rel,
            std::log2(rel));
  }
  int hfb = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&hfb, fbn.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  ctx->knn_fallback = hfb;  // diagnostics (gs_ctx_knn_fallback)
  GS_TRY(gs_knn_brute_list(ctx, dpts, sq, n, d, k, fb.get(), hfb, dnb, deps));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

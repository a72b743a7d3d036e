// gs_persist.cuh -- whole Sinkhorn sweeps in one persistent kernel for small one-pair fp64
// problems (BASELINE config 0: n = 2000, K = 30, 100 sweeps).
//
// Reference path: the sweep loop of sinkhorn_many / sinkhorn_single (proj/src/transport.cpp:
// 177-227) over HeatFilter::apply (heat.cpp:116-131) and SparseSymMatrix::multiply
// (sparse.cpp:85-99). At n = 2000 one Chebyshev step is ~25k multiply-adds: the graph-replayed
// per-step kernels (k_cheb_step_w1) are bound by the ~3.5 us a dependent kernel node costs, not
// by the work. Here one thread-block cluster of kPersistCluster CTAs runs every sweep:
//   * CTA r of the cluster owns rows [r R, (r + 1) R) of the filter's locality order, one thread
//     per row; its CSR slice lives in its shared memory in ELL order (entry u of the 32 rows of a
//     warp contiguous, so a warp's entry loads are conflict-free), its rows' a, M, N, V, W,
//     T_{k-1}, T_{k-2} and acc in registers;
//   * every CTA keeps a replica of the whole vector T (two buffers); a thread writes its row's T_k
//     into its own replica and pushes it with `st.async` (8 bytes, mbarrier complete_tx) into the
//     replicas of the CTAs whose rows read it (the owners of the row's neighbours), so a step needs
//     one __syncthreads and one wait on the CTA's own mbarrier for its halo bytes -- no cluster
//     barrier. The graph is symmetric, so CTAs that exchange rows stay within one step of each other
//     and two replica buffers suffice;
//   * the epilogues (W = N / max(psi, floor), V' = M / max(phi, floor), next T_0 = a x), the
//     positivity check, the L1 marginal error and the convergence / stagnation control run in the
//     same kernel; each CTA pushes its (min, max, error) partial to every CTA, which fold them in
//     rank order, so every CTA takes the same decision.
// Per row the fma chain, the recurrence, the acc update order (b_0/2 T_0, then fma(b_k, T_k, acc))
// and the epilogue arithmetic are those of k_cheb_step / finish_row_ops: v and w are bit-identical
// to the per-step kernels and to the oracle. Only the L1 error's summation order differs (a control
// input; k_finalize's order is not the oracle's either).
#pragma once

#include <cooperative_groups.h>

#include "gs_step.cuh"

namespace gsk {

constexpr int kPersistClusterMax = 16;  // CTAs per cluster at most (16: non-portable opt-in)
constexpr int kPersistMaxRows = 512;   // rows per CTA (one thread per row)
constexpr int kPersistMaxN = 8192;     // replica of T: 2 x n doubles per CTA

struct PersistArgs {
  int n, R, K, max_iter, no_abort;
  double tol, slack;
  const double* coeffs;  // b_0 .. b_K (device)
  const int* offs;
  const int* cols;
  const double* vals;
  const double* a;  // n (locality order)
  const double* M;
  const double* N;
  double* V0;  // V_s lives in V[s & 1] (sinkhorn_impl's convention)
  double* V1;
  double* W;
  const double* T0;  // T_0 = a V_1 of sweep 1's first apply
  double* thr;       // column state (P = 1)
  int* iters;
  int* conv;
  int* stag;
  int* final_sweep;
  double* err_out;
  gs_status* status;
  int knp_code;
};

__host__ __device__ constexpr int persist_rep_offset(int n) {
  return (64 + 2 * kPersistClusterMax * 4 * 8 + 68 * 4 + n + 15) & ~15;
}

__device__ __forceinline__ unsigned mapa_u32(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(unsigned addr, double v, unsigned mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(mbar)
               : "memory");
}
// the data pushed by st.async is visible to threads that observe the phase completion of the
// (own CTA's) mbarrier it signals: a CTA-scope acquire, no L1 invalidation
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* bar, unsigned parity) { mbar_wait(bar, parity); }

__global__ void __launch_bounds__(kPersistMaxRows, 1) k_sk_persist(const PersistArgs P) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int CL = (int)cl.num_blocks();  // CTAs of the cluster (= of the grid)
  const int R = P.R, n = P.n, K = P.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int r0 = rank * R;
  const int r1 = min(n, r0 + R);
  const int row = r0 + tid;
  const bool own = row < r1;
  extern __shared__ __align__(16) unsigned char psm[];
  // layout: bars[8] u64 | red[2][16][4] doubles | wmax[32], wbase[33] ints | flag[n] bytes |
  //         Rep[2][n] doubles | ELL values | ELL columns
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(psm);  // step[2], red[2]
  double* red = reinterpret_cast<double*>(psm + 64);
  int* wmax = reinterpret_cast<int*>(psm + 64 + 2 * kPersistClusterMax * 4 * 8);
  int* wbase = wmax + 32;
  int* halo = wbase + 33;
  unsigned char* flag = reinterpret_cast<unsigned char*>(halo + 3);
  double* Rep = reinterpret_cast<double*>(psm + persist_rep_offset(n));
  double* eval = Rep + 2 * n;
  // ---- setup: ELL slice, push targets, halo size, replica of T_0 ---------------------------------
  const int pb = own ? P.offs[row] : 0;
  const int deg = own ? P.offs[row + 1] - pb : 0;
  const int wd = __reduce_max_sync(0xffffffffu, deg);
  if (lane == 0) wmax[warp] = wd;
  for (int i = tid; i < n; i += blockDim.x) flag[i] = 0;
  if (tid == 0) halo[0] = 0;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < nwarps; ++w) {
      wbase[w] = acc;
      acc += 32 * wmax[w];
    }
    wbase[nwarps] = acc;
  }
  __syncthreads();
  const int ne = wbase[nwarps];
  int* ecol = reinterpret_cast<int*>(eval + ne);
  const int eb = wbase[warp] + lane;
  unsigned dst_mask = 0;  // CTAs whose rows read this row
  for (int u = 0; u < wd; ++u) {
    int c = 0;
    double v = 0.0;
    if (u < deg) {
      c = P.cols[pb + u];
      v = P.vals[pb + u];
      const int o = c / R;
      if (o != rank) {
        dst_mask |= 1u << o;
        flag[c] = 1;
      }
    }
    ecol[eb + u * 32] = c;
    eval[eb + u * 32] = v;
  }
  for (int i = tid; i < n; i += blockDim.x) Rep[i] = P.T0[i];  // T_0 of sweep 1, every row
  __syncthreads();
  {
    int cnt = 0;
    for (int i = tid; i < n; i += blockDim.x) cnt += flag[i];
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) atomicAdd(&halo[0], cnt);
  }
  __syncthreads();
  // every row of this CTA (pushed to itself) + the halo rows of other CTAs
  const unsigned halo_bytes = ((unsigned)halo[0] + (unsigned)(r1 > r0 ? r1 - r0 : 0)) * 8u;
  if (tid == 0) {
    for (int b = 0; b < 4; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {  // epochs 1 and 2 (step bars' phase 0), reductions 0 and 1
    mbar_expect_tx(&bars[1], halo_bytes);
    mbar_expect_tx(&bars[0], halo_bytes);
    mbar_expect_tx(&bars[2], CL * 3 * 8);
    mbar_expect_tx(&bars[3], CL * 3 * 8);
  }
  cl.sync();  // every CTA's barriers initialised before anyone pushes
  const unsigned rep_s = smem_u32(Rep), bar_s = smem_u32(bars), red_s = smem_u32(red);
  double ai = 0.0, mi = 0.0, ni = 0.0, vi = 0.0, wi = 0.0;
  if (own) {
    ai = P.a[row];
    mi = P.M[row];
    ni = P.N[row];
    vi = P.V1[row];  // V_1 (initial apply)
  }
  const double b0h = P.coeffs[0] / 2.0;
  double thr = P.thr[0];
  int stag = 0;
  int epoch = 0;  // data epoch e lives in Rep[e & 1]; epoch e >= 1 arrives on bars[e & 1]
  int redn = 0;   // reductions so far
  // publish this row's value of epoch e (own replica + pushes), then wait for the epoch's halo
  auto publish = [&](double t) {
    const int e = epoch + 1;
    const int b = e & 1;
    if (own) {
      unsigned m = dst_mask | (1u << rank);  // the own replica too: one completion mechanism
      while (m) {
        const int q = __ffs(m) - 1;
        m &= m - 1;
        st_async_f64(mapa_u32(rep_s + (unsigned)((b * n + row) * 8), q), t, mapa_u32(bar_s + b * 8, q));
      }
    }
    mbar_wait_cluster(&bars[b], (unsigned)(((e - 1) >> 1) & 1));
    if (tid == 0) mbar_expect_tx(&bars[b], halo_bytes);  // epoch e + 2 on this barrier
    epoch = e;
  };
  // (min, max, error) over the cluster, folded in rank order on every CTA
  auto reduce = [&](double mn, double mx, double er, double (&out)[3]) {
    const int slot = redn & 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      er = er + __shfl_xor_sync(0xffffffffu, er, o);
    }
    double* wpart = eval;  // not needed here: the warp partials go through red's spare lanes
    (void)wpart;
    __shared__ double wp[32][3];
    if (lane == 0) {
      wp[warp][0] = mn;
      wp[warp][1] = mx;
      wp[warp][2] = er;
    }
    __syncthreads();
    if (tid < CL) {  // thread q pushes this CTA's partial to CTA q
      double a = wp[0][0], b = wp[0][1], c = wp[0][2];
      for (int w = 1; w < nwarps; ++w) {
        a = fmin(a, wp[w][0]);
        b = fmax(b, wp[w][1]);
        c = c + wp[w][2];
      }
      const unsigned dst = red_s + (unsigned)(((slot * kPersistClusterMax + rank) * 4) * 8);
      const unsigned mb = mapa_u32(bar_s + (2 + slot) * 8, tid);
      st_async_f64(mapa_u32(dst, tid), a, mb);
      st_async_f64(mapa_u32(dst + 8, tid), b, mb);
      st_async_f64(mapa_u32(dst + 16, tid), c, mb);
    }
    mbar_wait_cluster(&bars[2 + slot], (unsigned)((redn >> 1) & 1));
    double a = INFINITY, b = 0.0, c = 0.0;
    for (int r = 0; r < CL; ++r) {
      const double* rr = red + (slot * kPersistClusterMax + r) * 4;
      a = fmin(a, rr[0]);
      b = fmax(b, rr[1]);
      c = r == 0 ? rr[2] : c + rr[2];
    }
    out[0] = a;
    out[1] = b;
    out[2] = c;
    __syncthreads();  // everybody has read red[slot] and wp
    if (tid == 0) mbar_expect_tx(&bars[2 + slot], CL * 3 * 8);  // reduction redn + 2
    ++redn;
  };
  // one K-step apply of the filter to the replicated T_0 (epoch `epoch`); returns p_K(L_s) T_0
  auto apply = [&]() -> double {
    double tp = own ? Rep[(epoch & 1) * n + row] : 0.0;
    double t2 = 0.0, acc = 0.0;
    for (int k = 1; k <= K; ++k) {
      const double* src = Rep + (epoch & 1) * n;
      double t = 0.0;
      if (own) {
        // 16 entries' loads in flight at once (predicated), then the fma chain in CSR order
        double y = 0.0;
        for (int u0 = 0; u0 < deg; u0 += 16) {
          double xv[16], vv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const bool in = u0 + j < deg;
            const int ei = eb + (in ? u0 + j : 0) * 32;
            vv[j] = eval[ei];
            xv[j] = src[ecol[ei]];
          }
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (u0 + j < deg) y = fma(vv[j], xv[j], y);
        }
        // recurrence and acc (finish_row_ops order)
        t = k == 1 ? y - tp : 2.0 * (y - tp) - t2;
        acc = k == 1 ? fma(P.coeffs[1], t, b0h * tp) : fma(P.coeffs[k], t, acc);
        t2 = tp;
        tp = t;
      }
      if (k < K) publish(t);
    }
    return acc;
  };
  int sweep = 0, status = 0, fail_sweep = 0, done = 0;
  double err = 0.0;
  for (sweep = 1; sweep <= P.max_iter; ++sweep) {
    // ---- psi = H(a V_s); W_s = N / max(psi, floor); T_0 = a W_s --------------------------------
    const double psi = apply();
    double mn = INFINITY, mx = 0.0, tn = 0.0;
    if (own) {
      mn = psi;
      wi = ni / fmax(psi, GS_FLOOR);
      tn = ai * wi;
      mx = fabs(tn);
    }
    publish(tn);
    double rd[3];
    reduce(mn, mx, 0.0, rd);
    if (!(rd[0] >= -thr)) {
      status = P.knp_code;
      break;
    }
    thr = P.slack * rd[1];
    // ---- phi = H(a W_s); err; V_{s+1} = M / max(phi, floor); T_0 = a V_{s+1} --------------------
    const double phi = apply();
    double er = 0.0, vnext = 0.0;
    mn = INFINITY;
    mx = 0.0;
    tn = 0.0;
    if (own) {
      mn = phi;
      er = fabs(vi * phi - mi);
      vnext = mi / fmax(phi, GS_FLOOR);
      tn = ai * vnext;
      mx = fabs(tn);
    }
    publish(tn);
    reduce(mn, mx, er, rd);
    if (!(rd[0] >= -thr)) {
      status = P.knp_code;
      break;
    }
    thr = P.slack * rd[1];
    err = rd[2];
    // ---- control (k_sk_control, one pair) -------------------------------------------------------
    done = err <= P.tol;
    if (!done) {
      stag = err > 0.5 ? stag + 1 : 0;
      if (!P.no_abort && !(stag < 50)) {
        status = ERRC_DISCONNECTED + 1;
        fail_sweep = sweep;
        break;
      }
    }
    if (done || sweep == P.max_iter) break;  // V_s, W_s are the results
    vi = vnext;
  }
  // ---- results in sinkhorn_impl's buffers ---------------------------------------------------------
  if (status == 0 && own) {
    ((sweep & 1) ? P.V1 : P.V0)[row] = vi;
    P.W[row] = wi;
  }
  if (rank == 0 && tid == 0) {
    if (status) {
      P.status->error = status;
      P.status->fail_pair = 0;
      P.status->fail_sweep = fail_sweep;
    } else {
      P.iters[0] = sweep;
      P.err_out[0] = err;
      P.conv[0] = done;
      P.final_sweep[0] = sweep;
    }
    P.stag[0] = stag;
    P.status->n_active = 0;
  }
  cl.sync();  // no CTA exits while another may still push into its shared memory
}

}  // namespace gsk

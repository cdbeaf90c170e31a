// rebk_csr.cu — persistent REBK kernel for sparse A (CSR + CSC twin), sm_100a.
//
// The reference keeps a CSR matrix and its CSC twin (matrix.py:46-58) and
// applies the four block products through scipy's sparsetools
// (solvers.py:283-295):
//   u = A_Jᵀ z      csr_matvec of the transposed CSC slice: per column j of J,
//                   a sequential sum over its nonzeros in row order;
//   z -= s (A_J u)  csc_matvec: row i accumulates over the columns of J in
//                   column order, then z_i - s*y_i;
//   r = A_I x       csr_matvec: per row, sequential over its columns;
//   x -= s (A_Iᵀ r) csc_matvec of the transposed CSR slice: column j
//                   accumulates over the rows of I in row order.
// Here every product is a GATHER (no atomics): per-block segment lists
// (built once per partition on the host) give each row of a column block
// its [lo, hi) range in the CSR arrays and each column of a row block its
// range in the CSC arrays.  Sums run in scipy's order with unfused
// multiply/add, so the iterates reproduce scipy bit for bit.
//
// Per iteration, 2 grid barriers (the dependency chain u -> z -> r -> x):
//   P(k): stop decision for k-1; z update of the owned rows (u_k) except rows
//         of I; for each row of I: r_i and its own z update (no cross-thread
//         read of z).
//   Q(k): x update of the owned columns (r_k); error partial; u_{k+1}.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rebk_device.cuh"
#include "rebk_internal.h"

namespace rebk {

// latency-bound gathers: run 1024 threads per SM (4x the dense kernels)
constexpr int kCsrThreads = 1024;
constexpr int kCsrWarps = kCsrThreads / 32;

// fixed-order CTA sum for kCsrThreads threads
__device__ __forceinline__ double csr_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kCsrWarps; ++w) s += red[w];
  __syncthreads();
  return s;
}

// in-order sum of the 32 lane values `prod` (lanes [0, cnt)) onto sum
__device__ __forceinline__ double ordered_lane_sum(double sum, double prod, int cnt) {
  if (cnt == 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, prod, j));
  } else {
    for (int j = 0; j < cnt; ++j) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, prod, j));
  }
  return sum;
}

__device__ __forceinline__ double madd(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));  // no FMA contraction: scipy's order and rounding
}

// Σ_{e in [lo,hi)} val[e] * vec[idx[e] - off] in index order, by one warp:
// lanes form the products in parallel (the gathers overlap), every lane then
// adds them in order, so all lanes hold the same, scipy-ordered sum.
__device__ __forceinline__ double warp_ordered_dot(const double* __restrict__ val, const int32_t* __restrict__ idx,
                                                   const double* vec, int off, int64_t lo, int64_t hi) {
  const int lane = threadIdx.x & 31;
  double sum = 0.0;
  constexpr int kPf = 8;  // chunks whose gathers are all in flight before the ordered adds
  if (hi - lo <= 32 * kPf) {
    double prod[kPf];
#pragma unroll
    for (int c = 0; c < kPf; ++c) {
      const int64_t e = lo + 32 * c + lane;
      prod[c] = e < hi ? __dmul_rn(val[e], __ldcg(vec + (idx[e] - off))) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < kPf; ++c) {
      const int64_t base = lo + 32 * c;
      if (base < hi) sum = ordered_lane_sum(sum, prod[c], (int)((hi - base) < 32 ? (hi - base) : 32));
    }
    return sum;
  }
  for (int64_t base = lo; base < hi; base += 32) {
    const int64_t e = base + lane;
    double prod = 0.0;
    if (e < hi) prod = __dmul_rn(val[e], __ldcg(vec + (idx[e] - off)));
    const int cnt = (int)((hi - base) < 32 ? (hi - base) : 32);
    sum = ordered_lane_sum(sum, prod, cnt);
  }
  return sum;
}

__global__ void __launch_bounds__(kCsrThreads) rebk_csr_kernel(CsrParams p) {
  // u and r staged per CTA: gathered straight from L2, the few dozen lines
  // of these short vectors are hammered by every thread of every SM (the z /
  // x updates are one gather per stored entry), which serialises on their L2
  // slices; one coalesced copy per CTA and gathers from shared memory instead
  extern __shared__ __align__(16) double s_vec[];
  double* s_u = s_vec;
  double* s_r = s_vec + p.su_cap;
  const bool st_u = p.su_cap > 0, st_r = p.sr_cap > 0;
  __shared__ double s_red[kCsrWarps];
  __shared__ double s_bcast[2];
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int64_t gtid = (int64_t)g * kCsrThreads + tid, gthreads = (int64_t)G * kCsrThreads;
  Control* ctl = p.ctl;
  if (*((volatile int32_t*)&ctl->done)) return;

  const int xq0 = split_rows(p.n, G, g), xq1 = split_rows(p.n, G, g + 1);
  const int zr0 = split_rows(p.m, G, g), zr1 = split_rows(p.m, G, g + 1);

  unsigned long long bar_target = 0;
  auto gsync = [&]() {
    bar_target += (unsigned long long)G;
    grid_barrier(&ctl->bar, bar_target);
  };
  const bool checking = p.stop_mode != 2;
  const bool oracle = p.stop_mode == 0;

  // Σ (x_j - x*_j)^2 over this CTA's columns by the warps [w0, 32) (fixed
  // order: per-thread strided sums, warp butterflies, the warp sums in warp
  // order); a named barrier of just those warps, so the others can be busy
  // with something else
  auto oracle_partial = [&](int w0) {
    const int T = (kCsrWarps - w0) * 32, t = tid - w0 * 32;
    if (t < 0) return;
    named_bar_sync(1, T);  // the group's own x updates are visible
    double acc = 0.0;
    for (int j = xq0 + t; j < xq1; j += T) {
      const double d = __ldcg(p.x + j) - __ldg(p.xs + j);
      acc = fma(d, d, acc);
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) s_red[warp] = acc;
    named_bar_sync(1, T);
    if (t == 0) {
      double sum = 0.0;
      for (int w = w0; w < kCsrWarps; ++w) sum += s_red[w];
      __stcg(p.errpart + g, sum);
    }
  };
  // ||Aᵀ(Ax - b + z)|| / scale (solvers.py:410-419) through csr/csc matvecs
  auto residual_partials = [&]() {
    for (int64_t i = gtid; i < p.m; i += gthreads) {
      double acc = 0.0;
      for (int64_t e = p.csr_ptr[i]; e < p.csr_ptr[i + 1]; ++e) acc = madd(acc, p.csr_val[e], __ldcg(p.x + p.csr_col[e]));
      double v = __dsub_rn(acc, __ldg(p.b + i));
      if (p.extended) v = __dadd_rn(v, __ldcg(p.z + i));
      __stcg(p.res + i, v);
    }
    gsync();
    double acc2 = 0.0;
    for (int j = xq0 + tid; j < xq1; j += kCsrThreads) {
      double gj = 0.0;
      for (int64_t e = p.csc_ptr[j]; e < p.csc_ptr[j + 1]; ++e) gj = madd(gj, p.csc_val[e], __ldcg(p.res + p.csc_row[e]));
      acc2 = fma(gj, gj, acc2);
    }
    const double s = csr_block_sum(acc2, s_red);
    if (tid == 0) __stcg(p.errpart + g, s);
  };
  auto decide = [&](int64_t k) -> bool {
    if (warp == 0) {
      double s = 0.0;
      for (int q = lane; q < G; q += 32) s += __ldcg(p.errpart + q);
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) s_bcast[0] = s;
    }
    __syncthreads();
    double err = sqrt(s_bcast[0]);
    if (!oracle) err = err / p.res_scale;
    const bool conv = check_stops(err, p.tol, p.nonfinite_stop);
    if (g == 0 && tid == 0) record_check(ctl, p.errs, p.errs_cap, p.record, err, p.tol, p.nonfinite_stop, k);
    __syncthreads();
    return conv;
  };
  // u_j = Σ_i A_ij z_i over CSC column j, for the column block of `pl`
  // (one warp per column; products gathered in parallel, summed in order)
  // items (columns of J, rows of I) go round-robin over CTAs first, then warps
  const int64_t gwarp = (int64_t)warp * G + g, gwarps = (int64_t)G * kCsrWarps;
  auto compute_u = [&](const Plan& pl) {
    for (int64_t j = pl.c_lo + gwarp; j < pl.c_hi; j += gwarps) {
      const double acc = warp_ordered_dot(p.csc_val, p.csc_row, p.z, 0, p.csc_ptr[j], p.csc_ptr[j + 1]);
      if (lane == 0) __stcg(p.u + (j - pl.c_lo), acc);
    }
  };

  // ---- L2 prefetch of the block data the coming phases read.  The phases
  // are chains of dependent loads (segment -> entries -> gathered vector); a
  // randomly sampled block comes from HBM (A and its copies are several times
  // L2), so every link of the chain costs a DRAM latency.  The block sequence
  // is known, and a block's data is a handful of contiguous ranges: while the
  // row sweep runs (most warps have no row of I), lane 0 of the last four
  // warps pulls the ranges of the phases that follow into L2 with bulk
  // prefetches; the chains then run on L2 hits.
  auto prefetch_range = [&](const void* base, int64_t lo_bytes, int64_t hi_bytes) {
    const int64_t a = lo_bytes & ~(int64_t)15, b = hi_bytes & ~(int64_t)15;  // stay inside the array
    const char* q = static_cast<const char*>(base) + a;
    for (int64_t left = b - a; left > 0; left -= (int64_t)1 << 20, q += (int64_t)1 << 20)
      bulk_prefetch_l2(q, (uint32_t)(left < ((int64_t)1 << 20) ? left : ((int64_t)1 << 20)));
  };
  // this CTA's even share of entries [lo, hi)
  auto share = [&](int64_t lo, int64_t hi, int64_t& a, int64_t& b) {
    a = lo + (hi - lo) * g / G;
    b = lo + (hi - lo) * (g + 1) / G;
  };
  // which: 0 = the x update of `cur` (row block copy); 1 = u of `nxt` (CSC
  // columns of its column block); 2 = the z update of `nxt` (column block
  // copy); 3 = the row sweep of `nxt` (CSR rows of its row block)
  auto prefetch_phase_data = [&](int which, const Plan& cur, const Plan* nxt) {
    if (which == 0) {
      const int64_t s0 = p.rseg_cta[(int64_t)cur.rb * (G + 1) + g], s1 = p.rseg_cta[(int64_t)cur.rb * (G + 1) + g + 1];
      if (s1 <= s0) return;
      prefetch_range(p.rseg_col, s0 * 4, s1 * 4);
      prefetch_range(p.rseg_ptr, s0 * 8, (s1 + 1) * 8);
      const int64_t e0 = p.rseg_ptr[s0], e1 = p.rseg_ptr[s1];
      prefetch_range(p.rval, e0 * 8, e1 * 8);
      prefetch_range(p.rrow, e0 * 4, e1 * 4);
    } else if (!nxt) {
      return;
    } else if (which == 1) {
      if (!p.extended) return;
      int64_t a, b;
      share(p.csc_ptr[nxt->c_lo], p.csc_ptr[nxt->c_hi], a, b);
      prefetch_range(p.csc_val, a * 8, b * 8);
      prefetch_range(p.csc_row, a * 4, b * 4);
    } else if (which == 2) {
      if (!p.extended) return;
      const int64_t s0 = p.cseg_cta[(int64_t)nxt->cb * (G + 1) + g], s1 = p.cseg_cta[(int64_t)nxt->cb * (G + 1) + g + 1];
      if (s1 <= s0) return;
      prefetch_range(p.cseg_row, s0 * 4, s1 * 4);
      prefetch_range(p.cseg_ptr, s0 * 8, (s1 + 1) * 8);
      const int64_t e0 = p.cseg_ptr[s0], e1 = p.cseg_ptr[s1];
      prefetch_range(p.cval, e0 * 8, e1 * 8);
      prefetch_range(p.ccol, e0 * 4, e1 * 4);
    } else {
      int64_t a, b;
      share(p.csr_ptr[nxt->r_lo], p.csr_ptr[nxt->r_hi], a, b);
      prefetch_range(p.csr_val, a * 8, b * 8);
      prefetch_range(p.csr_col, a * 4, b * 4);
    }
  };

  // phase counters only in profiling builds (-DREBK_KERNEL_PROF): at 1024
  // threads the kernel has 64 registers per thread, and keeping 8 live
  // 64-bit counters for a runtime flag made it spill
#ifdef REBK_KERNEL_PROF
  long long prof_acc[8];
  for (int i = 0; i < 8; ++i) prof_acc[i] = 0;
  long long prof_last = clock64();
#define PROF(i)                      \
  if (p.prof) {                      \
    const long long _t = clock64();  \
    prof_acc[i] += _t - prof_last;   \
    prof_last = _t;                  \
  }
#else
#define PROF(i)
#endif
  bool finished = false;
  if (p.k_begin == 1 && checking) {
    if (oracle) {
      oracle_partial(0);
      gsync();
    } else {
      residual_partials();
      gsync();
    }
    if (decide(0)) finished = true;
  }
  if (!finished && p.extended && p.k_begin <= p.k_end) {
    compute_u(p.plan[0]);
    gsync();
  }

  bool pending = false;
  int64_t pending_k = 0;
  for (int64_t k = p.k_begin; !finished && k <= p.k_end; ++k) {
    const Plan pl = p.plan[k - p.k_begin];
    const bool check_k = checking && (k % p.stride == 0);
    // ---- P(k)
    // u_k (complete since the last barrier) into shared memory; the loads fly
    // while warp 0 sums the error partials of the pending check
    if (p.extended && st_u)
      for (int c = tid; c < pl.c_hi - pl.c_lo; c += kCsrThreads) s_u[c] = __ldcg(p.u + c);
    if (pending && warp == 0) {  // (decide(), with its loads beside the copy's and one barrier for both)
      double sum = 0.0;
      for (int q = lane; q < G; q += 32) sum += __ldcg(p.errpart + q);
      for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      if (lane == 0) s_bcast[0] = sum;
    }
    if (pending || (p.extended && st_u)) __syncthreads();
    if (pending) {
      pending = false;
      double err = sqrt(s_bcast[0]);
      if (!oracle) err = err / p.res_scale;
      const bool conv = check_stops(err, p.tol, p.nonfinite_stop);
      if (g == 0 && tid == 0) record_check(ctl, p.errs, p.errs_cap, p.record, err, p.tol, p.nonfinite_stop, pending_k);
      if (conv) {
        finished = true;
        break;
      }
    }
    const double cs = pl.c_scale, rs = pl.r_scale;
    PROF(0);
    // The z update of the rows outside I (one thread per segment) and the row
    // sweep (one warp per row of I) are independent: when the CTA's rows of I
    // occupy only some warps, the other warps take all the segments and the
    // two run side by side
    const int nI = pl.r_hi - pl.r_lo;
    int nrw = nI > g ? (nI - g + G - 1) / G : 0;  // warps of this CTA with a row of I (rows: CTAs first, then warps)
    const bool split_p = p.extended && p.specialize && nrw <= kCsrWarps - 8;
    const int segT = split_p ? (kCsrWarps - nrw) * 32 : kCsrThreads;
    const int segt = split_p ? tid - nrw * 32 : tid;
    if (p.extended && segt >= 0) {
      const int64_t s0 = p.cseg_cta[(int64_t)pl.cb * (G + 1) + g];
      const int64_t s1 = p.cseg_cta[(int64_t)pl.cb * (G + 1) + g + 1];
      for (int64_t sg = s0 + segt; sg < s1; sg += segT) {
        const int i = p.cseg_row[sg];
        if (i >= pl.r_lo && i < pl.r_hi) continue;  // done by the row-sweep threads below
        const double zi = __ldcg(p.z + i);  // issued with the entry loads, not after the sum
        double acc = 0.0;
        const int64_t e1 = p.cseg_ptr[sg + 1];
        if (st_u)
          for (int64_t e = p.cseg_ptr[sg]; e < e1; ++e) acc = madd(acc, p.cval[e], s_u[p.ccol[e]]);
        else
          for (int64_t e = p.cseg_ptr[sg]; e < e1; ++e) acc = madd(acc, p.cval[e], __ldcg(p.u + p.ccol[e]));
        __stcg(p.z + i, __dsub_rn(zi, __dmul_rn(cs, acc)));
      }
    }
    PROF(1);
    // rows of I: one warp per row; r_i and the row's own z update
    for (int64_t i = pl.r_lo + gwarp; i < pl.r_hi; i += gwarps) {
      double ax = 0.0, au = 0.0;
      const double bi = __ldg(p.b + i);
      const double zi = p.extended ? __ldcg(p.z + i) : 0.0;  // nobody else writes z_i of a row of I in P(k)
      const int64_t lo = p.csr_ptr[i], hi = p.csr_ptr[i + 1];
      constexpr int kPf = 4;  // a row's gathers all in flight, then the ordered adds
      int64_t base = lo;
      while (base < hi) {
        double px[kPf], pu[kPf];
#pragma unroll
        for (int c = 0; c < kPf; ++c) {
          const int64_t e = base + 32 * c + lane;
          px[c] = 0.0;
          pu[c] = 0.0;
          if (e < hi) {
            const int col = p.csr_col[e];
            const double a = p.csr_val[e];
            px[c] = __dmul_rn(a, __ldcg(p.x + col));
            if (p.extended && col >= pl.c_lo && col < pl.c_hi)
              pu[c] = __dmul_rn(a, st_u ? s_u[col - pl.c_lo] : __ldcg(p.u + (col - pl.c_lo)));
          }
        }
#pragma unroll
        for (int c = 0; c < kPf; ++c) {
          const int64_t b0 = base + 32 * c;
          if (b0 < hi) {
            const int cnt = (int)((hi - b0) < 32 ? (hi - b0) : 32);
            ax = ordered_lane_sum(ax, px[c], cnt);
            // entries outside J contribute +0.0, an exact no-op on the running sum
            if (p.extended) au = ordered_lane_sum(au, pu[c], cnt);
          }
        }
        base += 32 * kPf;
      }
      if (lane == 0) {
        double rv = __dsub_rn(ax, bi);
        if (p.extended) {
          const double zn = __dsub_rn(zi, __dmul_rn(cs, au));
          __stcg(p.z + i, zn);
          rv = __dadd_rn(rv, zn);
        }
        __stcg(p.r + (i - pl.r_lo), rv);
      }
    }
    if (p.l2_prefetch && lane == 0 && warp >= kCsrWarps - 4)
      prefetch_phase_data(warp - (kCsrWarps - 4), pl, k < p.k_end ? &p.plan[k + 1 - p.k_begin] : nullptr);
    PROF(2);
    gsync();
    PROF(3);
    // ---- Q(k): the x update (one thread per segment), the error partial of
    // a check, and u_{k+1} (one warp per column of the next column block, from
    // z_k) — u does not depend on x, so when its columns occupy only some of
    // the CTA's warps the others do the x update and the check beside it
    const Plan* nxt = (p.extended && k < p.k_end) ? &p.plan[k + 1 - p.k_begin] : nullptr;
    int ncw = 0;
    if (nxt) {
      const int nJn = nxt->c_hi - nxt->c_lo;
      ncw = nJn > g ? (nJn - g + G - 1) / G : 0;
    }
    const bool split_q = p.specialize && ncw > 0 && ncw <= kCsrWarps - 8 && (!check_k || oracle);
    {
      const int64_t s0 = p.rseg_cta[(int64_t)pl.rb * (G + 1) + g];
      const int64_t s1 = p.rseg_cta[(int64_t)pl.rb * (G + 1) + g + 1];
      if (st_r) {
        for (int c = tid; c < pl.r_hi - pl.r_lo; c += kCsrThreads) s_r[c] = __ldcg(p.r + c);
        __syncthreads();
      }
      const int xT = split_q ? (kCsrWarps - ncw) * 32 : kCsrThreads;
      const int xt = split_q ? tid - ncw * 32 : tid;
      if (xt >= 0)
        for (int64_t sg = s0 + xt; sg < s1; sg += xT) {
          const int j = p.rseg_col[sg];
          // step_dsbgs: only x[J] moves (solvers.py:378-379)
          if (p.dsbgs && (j < pl.c_lo || j >= pl.c_hi)) continue;
          const double xj = __ldcg(p.x + j);
          double acc = 0.0;
          const int64_t e1 = p.rseg_ptr[sg + 1];
          if (st_r)
            for (int64_t e = p.rseg_ptr[sg]; e < e1; ++e) acc = madd(acc, p.rval[e], s_r[p.rrow[e]]);
          else
            for (int64_t e = p.rseg_ptr[sg]; e < e1; ++e) acc = madd(acc, p.rval[e], __ldcg(p.r + p.rrow[e]));
          __stcg(p.x + j, __dsub_rn(xj, __dmul_rn(rs, acc)));
        }
    }
    if (split_q) {
      if (warp < ncw) {
        compute_u(*nxt);
      } else if (check_k) {
        oracle_partial(ncw);
      }
      if (check_k) {  // uniform across the CTA
        pending = true;
        pending_k = k;
      }
      PROF(4);
    } else {
      __syncthreads();
      PROF(4);
      if (check_k) {
        if (oracle) {
          oracle_partial(0);
          pending = true;
          pending_k = k;
        } else {
          gsync();
          residual_partials();
          gsync();
          if (decide(k)) {
            finished = true;
            break;
          }
        }
      }
      PROF(5);
      if (nxt) compute_u(*nxt);
    }
    PROF(6);
    gsync();
    PROF(7);
  }

  if (!finished) {
    if (pending) {
      if (decide(pending_k)) finished = true;  // errpart was published before the loop's last barrier
    }
    if (!finished && p.k_end == p.max_iters) {
      if (checking && (p.max_iters % p.stride) != 0) {
        if (oracle) {
          oracle_partial(0);
          gsync();
        } else {
          residual_partials();
          gsync();
        }
        decide(p.max_iters);
      }
      if (g == 0 && tid == 0) {
        if (!ctl->converged) ctl->iters = p.max_iters;
        ctl->done = 1;
      }
    }
  }
#ifdef REBK_KERNEL_PROF
  if (p.prof && tid == 0)
    for (int i = 0; i < 8; ++i) p.prof[g * 16 + i] = prof_acc[i];
#endif
#undef PROF
}

static cudaError_t set_csr_attrs() {
  static int configured_device = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || configured_device == dev) return e;
  e = cudaFuncSetAttribute(rebk_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCsrStageBytesMax);
  if (e == cudaSuccess) configured_device = dev;
  return e;
}

cudaError_t launch_csr(const CsrParams& p, int G, cudaStream_t stream) {
  cudaError_t e = set_csr_attrs();
  if (e != cudaSuccess) return e;
  CsrParams pc = p;
  void* args[] = {&pc};
  const size_t smem = sizeof(double) * ((size_t)p.su_cap + (size_t)p.sr_cap);
  return cudaLaunchCooperativeKernel((const void*)rebk_csr_kernel, dim3(G), dim3(kCsrThreads), args, smem, stream);
}

cudaError_t csr_kernel_occupancy(size_t smem_bytes, int* blocks_per_sm) {
  cudaError_t e = set_csr_attrs();
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, rebk_csr_kernel, kCsrThreads, smem_bytes);
}

}  // namespace rebk

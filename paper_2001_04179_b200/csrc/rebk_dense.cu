// rebk_dense.cu — persistent fp64 REBK kernel for dense A on B200 (sm_100a).
//
// One launch runs a whole chunk of REBK iterations (solvers.py:450-458 loop,
// step_rebk solvers.py:324-337) without returning to the host.  Work split,
// fixed for the whole run:
//   * CTA g owns rows [zr0, zr1) of z   (column sweep:  u = A_JᵀZ, z -= s A_J u)
//   * CTA g owns cols [xq0, xq1) of x   (row sweep:     r = A_I x - b_I + z_I,
//                                                       x -= s A_Iᵀ r)
// Per iteration (5 phases, 4 grid barriers):
//   P1  upart[:,g] = A[zr, J]ᵀ z[zr]                          (col tile, TMA-staged)
//   P2  u = Σ_g upart  (entries spread over CTAs, fixed order) (+ pending stop decision)
//   P3  z[zr] -= s_J · A[zr, J] u ;  rpart[:,g] = A[I, xq] x[xq] (row tile, TMA-staged)
//   P4  r = ((Σ_g rpart) - b_I) + z_I                           (+ prefetch next col tile)
//   P5  x[xq] -= s_I · A[I, xq]ᵀ r ; err partial Σ(x - x*)²
// Both block tiles are read from HBM once: cp.async.bulk copies land them in
// shared memory one or more barriers before they are needed, and the second
// product of each sweep re-reads them from shared memory.  All reductions use
// a fixed order, so runs replay bit for bit (test_solvers.py:452-459).
#include <cuda_runtime.h>
#include <stdint.h>

#include "philox.h"
#include "rebk_device.cuh"
#include "rebk_internal.h"

namespace rebk {

// stage rows [row0, row0+R) x cols [col0, col0+C) of A into tile (ld doubles)
// with one bulk copy per row; bytes rounded up to 16 (the host guarantees the
// extra element is inside the allocation).  Issued by warp 0.
__device__ __forceinline__ void stage_tile(double* tile, int ld, const double* A, int64_t lda,
                                           int row0, int R, int col0, int C, uint64_t* bar) {
  if (threadIdx.x >= 32) return;
  const uint32_t row_bytes = (uint32_t)(((C + 1) & ~1) * 8);
  if (R <= 0 || C <= 0) {
    if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, 0);
    return;
  }
  if (threadIdx.x == 0) {
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, row_bytes * (uint32_t)R);
  }
  __syncwarp();
  for (int r = threadIdx.x; r < R; r += 32)
    bulk_g2s(tile + (int64_t)r * ld, A + (int64_t)(row0 + r) * lda + col0, row_bytes, bar);
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(kThreads, 1) rebk_dense_kernel(DenseParams p) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t mbar[2];  // 0: column tile, 1: row tile
  __shared__ double s_bcast[2];

  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  Control* ctl = p.ctl;
  if (*((volatile int32_t*)&ctl->done)) return;

  const int zr0 = split_rows(p.m, G, g), zr1 = split_rows(p.m, G, g + 1);
  const int xq0 = split_even(p.n, G, g), xq1 = split_even(p.n, G, g + 1);
  const int nR = zr1 - zr0, nC = xq1 - xq0;

  double* s_ct = sm + p.ct_off;
  double* s_rt = sm + p.rt_off;
  double* s_x = sm + p.vec_off;
  double* s_xs = s_x + p.nC_max;
  double* s_z = s_xs + p.nC_max;
  double* s_u = s_z + p.nR_max;
  double* s_r = s_u + p.nJ_max;
  double* s_red = s_r + p.nI_max;

  for (int c = tid; c < nC; c += kThreads) {
    s_x[c] = __ldcg(p.x + xq0 + c);
    s_xs[c] = p.xs ? __ldg(p.xs + xq0 + c) : 0.0;
  }
  if (p.extended)
    for (int r = tid; r < nR; r += kThreads) s_z[r] = __ldcg(p.z + zr0 + r);
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  unsigned long long bar_target = 0;
  auto gsync = [&]() {
    bar_target += (unsigned long long)G;
    grid_barrier(&ctl->bar, bar_target);
  };

  const bool checking = p.stop_mode != 2;
  const bool oracle = p.stop_mode == 0;

  // error partial of the current x slice, to errpart[g]
  auto oracle_partial = [&]() {
    double acc = 0.0;
    for (int c = tid; c < nC; c += kThreads) {
      const double d = s_x[c] - s_xs[c];
      acc = fma(d, d, acc);
    }
    const double s = block_sum(acc, s_red);
    if (tid == 0) __stcg(p.errpart + g, s);
  };
  // residual proxy ||Aᵀ(Ax - b + z)|| / scale, partial to errpart[g]
  // (solvers.py:410-419); needs the full x in global memory.
  auto residual_partials = [&]() {
    for (int c = tid; c < nC; c += kThreads) __stcg(p.x + xq0 + c, s_x[c]);
    gsync();
    const double* Arows = p.A + (int64_t)zr0 * p.lda;
    tile_rowdot<LdNC, LdCG>(Arows, p.lda, nR, p.n, p.x, [&](int r, double acc) {
      double v = acc - __ldg(p.b + zr0 + r);
      if (p.extended) v += s_z[r];
      __stcg(p.res + zr0 + r, v);
    });
    gsync();
    double acc = 0.0;
    tile_colsum<LdNC, LdCG>(p.A + xq0, p.lda, p.m, nC, p.res, s_red, [&](int, double gc) {
      acc = fma(gc, gc, acc);
    });
    const double s = block_sum(acc, s_red);
    if (tid == 0) __stcg(p.errpart + g, s);
  };
  // all CTAs: reduce errpart in fixed order and decide (identical everywhere)
  auto decide = [&](int64_t k) -> bool {
    if (warp == 0) {
      const double s = warp_sum_cg(p.errpart, G);
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

  bool ct_pending = false, rt_pending = false;
  uint32_t ct_par = 0, rt_par = 0;
  auto wait_ct = [&]() {
    if (ct_pending) {
      mbar_wait(&mbar[0], ct_par);
      ct_par ^= 1u;
      ct_pending = false;
    }
  };
  auto wait_rt = [&]() {
    if (rt_pending) {
      mbar_wait(&mbar[1], rt_par);
      rt_par ^= 1u;
      rt_pending = false;
    }
  };
  auto issue_ct = [&](const Plan& pl) {
    if (!p.stage_ct) return;
    stage_tile(s_ct, p.ct_ld, p.A, p.lda, zr0, nR, pl.c_lo, pl.c_hi - pl.c_lo, &mbar[0]);
    ct_pending = true;
  };
  auto issue_rt = [&](const Plan& pl) {
    if (!p.stage_rt) return;
    stage_tile(s_rt, p.rt_ld, p.A, p.lda, pl.r_lo, pl.r_hi - pl.r_lo, xq0, nC, &mbar[1]);
    rt_pending = true;
  };

  long long prof_acc[16];
  for (int i = 0; i < 16; ++i) prof_acc[i] = 0;
  long long prof_last = clock64();
#define PROF(i)                                  \
  if (p.prof) {                                  \
    const long long _t = clock64();              \
    prof_acc[i] += _t - prof_last;               \
    prof_last = _t;                              \
  }
  bool finished = false;
  // ---- check(0) (solvers.py:444)
  if (p.k_begin == 1 && checking) {
    if (oracle) {
      oracle_partial();
      gsync();
    } else {
      residual_partials();
      gsync();
    }
    if (decide(0)) finished = true;
  }

  bool pending = false;
  int64_t pending_k = 0;
  int64_t k = p.k_begin;
  if (!finished && p.extended && p.k_begin <= p.k_end) issue_ct(p.plan[0]);

  for (; !finished && k <= p.k_end; ++k) {
    const Plan pl = p.plan[k - p.k_begin];
    const int cl = pl.c_lo, nJ = pl.c_hi - pl.c_lo;
    const int rl = pl.r_lo, nI = pl.r_hi - pl.r_lo;
    const bool check_k = checking && (k % p.stride == 0);

    __syncthreads();  // previous readers of the row tile are done
    issue_rt(pl);
    PROF(0);

    if (p.extended) {
      // P1: partial u over owned rows
      const double* ct = p.stage_ct ? s_ct : p.A + (int64_t)zr0 * p.lda + cl;
      const int64_t ctld = p.stage_ct ? p.ct_ld : p.lda;
      wait_ct();
      PROF(1);
      auto up_epi = [&](int c, double val) { __stcg(p.upart + (int64_t)c * G + g, val); };
      if (p.stage_ct)
        tile_colsum<LdShared, LdShared>(ct, ctld, nR, nJ, s_z, s_red, up_epi);
      else
        tile_colsum<LdNC, LdShared>(ct, ctld, nR, nJ, s_z, s_red, up_epi);
      PROF(2);
      gsync();
      PROF(3);
      // P2: pending stop decision, then u = Σ_g upart
      if (pending) {
        pending = false;
        if (decide(pending_k)) {
          finished = true;
          break;
        }
      }
      for (int e = g * kWarps + warp; e < nJ; e += G * kWarps) {
        const double s = warp_sum_cg(p.upart + (int64_t)e * G, G);
        if (lane == 0) __stcg(p.u + e, s);
      }
      PROF(4);
      gsync();
      PROF(5);
      // P3a: z[zr] -= s_J · A[zr, J] u
      for (int c = tid; c < nJ; c += kThreads) s_u[c] = __ldcg(p.u + c);
      __syncthreads();
      const double cs = pl.c_scale;
      auto z_epi = [&](int r, double acc) {
        const double zn = s_z[r] - cs * acc;
        s_z[r] = zn;
        __stcg(p.z + zr0 + r, zn);
      };
      if (p.stage_ct)
        tile_rowdot<LdShared, LdShared>(ct, ctld, nR, nJ, s_u, z_epi);
      else
        tile_rowdot<LdNC, LdShared>(ct, ctld, nR, nJ, s_u, z_epi);
    }
    PROF(6);
    // P3b: partial r over owned columns
    {
      const double* rt = p.stage_rt ? s_rt : p.A + (int64_t)rl * p.lda + xq0;
      const int64_t rtld = p.stage_rt ? p.rt_ld : p.lda;
      wait_rt();
      PROF(7);
      auto rp_epi = [&](int r, double acc) { __stcg(p.rpart + (int64_t)r * G + g, acc); };
      if (p.stage_rt)
        tile_rowdot<LdShared, LdShared>(rt, rtld, nI, nC, s_x, rp_epi);
      else
        tile_rowdot<LdNC, LdShared>(rt, rtld, nI, nC, s_x, rp_epi);
    }
    PROF(8);
    gsync();
    PROF(9);
    // P4: (pending decision for row-only algorithms), r = ((Σ rpart) - b_I) + z_I
    if (!p.extended && pending) {
      pending = false;
      if (decide(pending_k)) {
        finished = true;
        break;
      }
    }
    if (p.extended && k < p.k_end) issue_ct(p.plan[k + 1 - p.k_begin]);
    for (int e = g * kWarps + warp; e < nI; e += G * kWarps) {
      const double s = warp_sum_cg(p.rpart + (int64_t)e * G, G);
      if (lane == 0) {
        double rv = s - __ldg(p.b + rl + e);
        if (p.extended) rv += __ldcg(p.z + rl + e);
        __stcg(p.r + e, rv);
      }
    }
    PROF(10);
    gsync();
    PROF(11);
    // P5: x[xq] -= s_I · A[I, xq]ᵀ r
    for (int c = tid; c < nI; c += kThreads) s_r[c] = __ldcg(p.r + c);
    __syncthreads();
    {
      const double* rt = p.stage_rt ? s_rt : p.A + (int64_t)rl * p.lda + xq0;
      const int64_t rtld = p.stage_rt ? p.rt_ld : p.lda;
      const double rs = pl.r_scale;
      // step_dsbgs: only the sampled column block's coordinates move
      // (x[J] -= s_ij A[I, J]^T r, solvers.py:378-379)
      auto x_epi = [&](int c, double acc) {
        if (!p.dsbgs || (xq0 + c >= cl && xq0 + c < cl + nJ)) s_x[c] = s_x[c] - rs * acc;
      };
      if (p.stage_rt)
        tile_colsum<LdShared, LdShared>(rt, rtld, nI, nC, s_r, s_red, x_epi);
      else
        tile_colsum<LdNC, LdShared>(rt, rtld, nI, nC, s_r, s_red, x_epi);
    }
    __syncthreads();
    PROF(12);
    if (check_k) {
      if (oracle) {
        oracle_partial();
        pending = true;
        pending_k = k;
      } else {
        residual_partials();
        gsync();
        if (decide(k)) {
          finished = true;
          ++k;
          break;
        }
      }
    }
  }

  if (!finished) {
    if (pending) {
      gsync();
      if (decide(pending_k)) finished = true;
    }
    if (!finished && p.k_end == p.max_iters) {
      // for-else branch of run(): a final check when max_iters is off-stride
      if (checking && (p.max_iters % p.stride) != 0) {
        if (oracle) {
          oracle_partial();
        } else {
          residual_partials();
        }
        gsync();
        decide(p.max_iters);
      }
      if (g == 0 && tid == 0) {
        if (!ctl->converged) ctl->iters = p.max_iters;
        ctl->done = 1;
      }
    }
  }
  if (p.prof && tid == 0)
    for (int i = 0; i < 16; ++i) p.prof[g * 16 + i] = prof_acc[i];
#undef PROF
  // write back the owned x slice; drain any bulk copy still in flight
  for (int c = tid; c < nC; c += kThreads) __stcg(p.x + xq0 + c, s_x[c]);
  if (tid == 0) {
    wait_ct();
    wait_rt();
  }
  __syncthreads();
}

static cudaError_t set_smem_attr() {
  static int configured_device = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured_device == dev) return cudaSuccess;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  // leave room for the kernel's static shared memory (mbarriers, broadcast)
  e = cudaFuncSetAttribute(rebk_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
  if (e == cudaSuccess) configured_device = dev;
  return e;
}

cudaError_t launch_dense(const DenseParams& p, int G, size_t smem_bytes, cudaStream_t stream) {
  cudaError_t e = set_smem_attr();
  if (e != cudaSuccess) return e;
  DenseParams pc = p;
  void* args[] = {&pc};
  return cudaLaunchCooperativeKernel((const void*)rebk_dense_kernel, dim3(G), dim3(kThreads), args,
                                     smem_bytes, stream);
}

cudaError_t dense_kernel_occupancy(size_t smem_bytes, int* blocks_per_sm) {
  cudaError_t e = set_smem_attr();
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, rebk_dense_kernel, kThreads,
                                                       smem_bytes);
}

// ------------------------------------------------------------------ sampler
// WeightedSampler.sample (sampling.py:137-145): v = u * total, index =
// #{cum <= v} (searchsorted side="right"), clamped to nb-1.
__device__ __forceinline__ int sample_block(const double* cum, int nb, double total, double u) {
  const double v = __dmul_rn(u, total);
  int lo = 0, hi = nb;  // first index with cum[idx] > v
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(cum + mid) <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < nb - 1 ? lo : nb - 1;
}

__device__ __forceinline__ uint64_t philox_word(uint64_t d, uint64_t k0, uint64_t k1) {
  const u64x4 blk = philox_block(d >> 2, k0, k1);
  return blk.v[d & 3];
}

__global__ void sample_plan_kernel(SampleParams sp, int64_t k0, int64_t count, Plan* plan,
                                   int32_t* picks_out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  const int64_t k = k0 + idx;  // 1-based iteration
  int j = -1, i;
  if (sp.picks) {
    j = sp.picks[2 * (k - 1)];
    i = sp.picks[2 * (k - 1) + 1];
  } else if (sp.dsbgs) {
    // step_dsbgs (solvers.py:371-375): column block from the column sampler
    // (draw 2(k-1)), then the row block from that column's conditional
    // sampler over its nonzero submatrices (draw 2k-1)
    const uint64_t dc = sp.draw_offset + 2ull * (uint64_t)(k - 1);
    const uint64_t wc = philox_word(dc, sp.key0, sp.key1), wr = philox_word(dc + 1, sp.key0, sp.key1);
    j = sample_block(sp.col_cum, sp.n_col_blocks, sp.col_total, u64_to_unit_double(wc));
    const int64_t o0 = sp.d_off[j], o1 = sp.d_off[j + 1];
    const int c = sample_block(sp.d_cum + o0, (int)(o1 - o0), sp.d_total[j], u64_to_unit_double(wr));
    i = sp.d_alive[o0 + c];
  } else {
    const uint64_t dc = sp.draw_offset + 2ull * (uint64_t)(k - 1);
    const uint64_t dr = dc + 1;
    uint64_t wc, wr;
    if ((dc >> 2) == (dr >> 2)) {
      const u64x4 blk = philox_block(dc >> 2, sp.key0, sp.key1);
      wc = blk.v[dc & 3];
      wr = blk.v[dr & 3];
    } else {
      wc = philox_word(dc, sp.key0, sp.key1);
      wr = philox_word(dr, sp.key0, sp.key1);
    }
    if (sp.extended) j = sample_block(sp.col_cum, sp.n_col_blocks, sp.col_total, u64_to_unit_double(wc));
    i = sample_block(sp.row_cum, sp.n_row_blocks, sp.row_total, u64_to_unit_double(wr));
  }
  if (plan) {
    Plan pl;
    if (sp.dsbgs) {
      pl.c_lo = (int32_t)sp.col_ptr[j];
      pl.c_hi = (int32_t)sp.col_ptr[j + 1];
      pl.c_scale = 0.0;
    } else if (sp.extended) {
      pl.c_lo = (int32_t)sp.col_ptr[j];
      pl.c_hi = (int32_t)sp.col_ptr[j + 1];
      pl.c_scale = sp.col_scale[j];
    } else {
      pl.c_lo = pl.c_hi = 0;
      pl.c_scale = 0.0;
    }
    pl.r_lo = (int32_t)sp.row_ptr[i];
    pl.r_hi = (int32_t)sp.row_ptr[i + 1];
    pl.r_scale = sp.dsbgs ? sp.d_scale[(int64_t)i * sp.n_col_blocks + j] : sp.row_scale[i];
    pl.cb = j;
    pl.rb = i;
    pl.pad0 = pl.pad1 = 0;
    plan[idx] = pl;
  }
  if (picks_out) {
    picks_out[2 * idx] = j;
    picks_out[2 * idx + 1] = i;
  }
}

cudaError_t launch_sample_plan(const SampleParams& sp, int64_t k0, int64_t count, Plan* plan,
                               int32_t* picks_out, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int tb = 256;
  const int64_t nblk = (count + tb - 1) / tb;
  sample_plan_kernel<<<(unsigned)nblk, tb, 0, stream>>>(sp, k0, count, plan, picks_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------- block norms
// ||A_block||_F^2 for contiguous row (axis 0) or column (axis 1) blocks
// (matrix.py:170-189), one CTA per block, fixed-order reduction.
__global__ void block_norms_kernel(const double* A, int64_t lda, int64_t m, int64_t n, int axis,
                                   const int64_t* ptr, double* out) {
  __shared__ double red[kWarps];
  const int64_t b = blockIdx.x;
  const int64_t lo = ptr[b], hi = ptr[b + 1];
  double acc = 0.0;
  if (axis == 0) {
    for (int64_t r = lo; r < hi; ++r)
      for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
        const double a = __ldg(A + r * lda + c);
        acc = fma(a, a, acc);
      }
  } else {
    const int64_t w = hi - lo;
    for (int64_t e = threadIdx.x; e < m * w; e += blockDim.x) {
      const double a = __ldg(A + (e / w) * lda + lo + e % w);
      acc = fma(a, a, acc);
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    out[b] = s;
  }
}

// fp32 storage (multi-RHS contexts): squares accumulated in fp64.  Each block
// is cut into kNormChunks row chunks (grid.y) so that a handful of wide
// blocks still fills the GPU; chunk partials part[b * kNormChunks + q] are
// summed in chunk order by block_norms_finish (fixed order: runs replay).
constexpr int kNormChunks = 32;
__global__ void block_norms_f32_kernel(const float* A, int64_t lda, int64_t m, int64_t n, int axis,
                                       const int64_t* ptr, double* part) {
  __shared__ double red[kWarps];
  const int64_t b = blockIdx.x;
  const int q = blockIdx.y;
  const int64_t lo = ptr[b], hi = ptr[b + 1];
  // rows of this chunk: axis 0 -> rows of the block, axis 1 -> all rows of A
  const int64_t R0 = axis == 0 ? lo : 0, R1 = axis == 0 ? hi : m;
  const int64_t r0 = R0 + (R1 - R0) * q / kNormChunks, r1 = R0 + (R1 - R0) * (q + 1) / kNormChunks;
  const int64_t c0 = axis == 0 ? 0 : lo, c1 = axis == 0 ? n : hi;
  double acc = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const float* row = A + r * lda;
    for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
      const double a = (double)__ldg(row + c);
      acc = fma(a, a, acc);
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part[b * kNormChunks + q] = s;
  }
}
__global__ void block_norms_finish(const double* part, int64_t nb, double* out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  double s = 0.0;
  for (int q = 0; q < kNormChunks; ++q) s += part[b * kNormChunks + q];
  out[b] = s;
}

// part_dev: scratch of nb * block_norms_f32_scratch() doubles
int64_t block_norms_f32_scratch() { return kNormChunks; }
cudaError_t launch_block_norms_f32(const float* A, int64_t lda, int64_t m, int64_t n, int axis, int64_t nb,
                                   const int64_t* ptr_dev, double* part_dev, double* out_dev, cudaStream_t stream) {
  if (nb <= 0) return cudaSuccess;
  block_norms_f32_kernel<<<dim3((unsigned)nb, kNormChunks), kThreads, 0, stream>>>(A, lda, m, n, axis, ptr_dev, part_dev);
  block_norms_finish<<<(unsigned)((nb + 127) / 128), 128, 0, stream>>>(part_dev, nb, out_dev);
  return cudaGetLastError();
}

cudaError_t launch_block_norms(const double* A, int64_t lda, int64_t m, int64_t n, int axis, int64_t nb,
                               const int64_t* ptr_dev, double* out_dev, cudaStream_t stream) {
  if (nb <= 0) return cudaSuccess;
  block_norms_kernel<<<(unsigned)nb, kThreads, 0, stream>>>(A, lda, m, n, axis, ptr_dev, out_dev);
  return cudaGetLastError();
}

}  // namespace rebk

namespace rebk {
// ---------------------------------------------------------- residual check
// The residual_proxy stopping rule of run() (solvers.py:410-421) as stand-
// alone kernels, for the clustered / split / streaming dense kernels, which
// run the iterations in chunks of check_stride between these checks:
//   res = A x - b (+ z),  g = Aᵀ res,  err = ||g|| / (||A||_F ||b||).
// Fixed-order reductions (warp per row; per-column partials over row chunks
// summed in chunk order), so a run replays bit for bit.
namespace {
constexpr int kResChunk = 256;  // rows per partial of Aᵀ res

__global__ void __launch_bounds__(256) k_res_rows(const double* __restrict__ A, int64_t lda, int m, int n,
                                                  const double* __restrict__ x, const double* __restrict__ b,
                                                  const double* __restrict__ z, const Control* ctl,
                                                  double* __restrict__ res) {
  if (*((volatile const int32_t*)&ctl->done)) return;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= m) return;
  const double* row = A + (int64_t)r * lda;
  double acc = 0.0;
  for (int c = lane; c < n; c += 32) acc = fma(__ldg(row + c), __ldcg(x + c), acc);
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) res[r] = acc - __ldg(b + r) + (z ? __ldcg(z + r) : 0.0);
}

__global__ void __launch_bounds__(256) k_res_cols(const double* __restrict__ A, int64_t lda, int m, int n,
                                                  const double* __restrict__ res, const Control* ctl,
                                                  double* __restrict__ part) {
  if (*((volatile const int32_t*)&ctl->done)) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x, chunk = blockIdx.y;
  if (c >= n) return;
  const int r0 = chunk * kResChunk, r1 = min(m, r0 + kResChunk);
  double acc = 0.0;
  for (int r = r0; r < r1; ++r) acc = fma(__ldg(A + (int64_t)r * lda + c), __ldcg(res + r), acc);
  part[(int64_t)chunk * n + c] = acc;
}

__global__ void __launch_bounds__(256) k_res_norm(int n, int nchunks, const double* __restrict__ part, Control* ctl,
                                                  double* __restrict__ colsq) {
  if (*((volatile const int32_t*)&ctl->done)) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double g = 0.0;
  for (int q = 0; q < nchunks; ++q) g += part[(int64_t)q * n + c];
  colsq[c] = g * g;
}

__global__ void __launch_bounds__(1024) k_res_decide(int n, const double* __restrict__ colsq, double scale, double tol,
                                                     int32_t nonfinite_stop, int32_t record, double* errs,
                                                     int64_t errs_cap, int64_t k, Control* ctl) {
  __shared__ double red[32];
  if (*((volatile const int32_t*)&ctl->done)) return;
  double acc = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) acc += colsq[c];
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    record_check(ctl, errs, errs_cap, record, sqrt(s) / scale, tol, nonfinite_stop, k);
  }
}
}  // namespace

cudaError_t launch_residual_check(const double* A, int64_t lda, int m, int n, const double* x, const double* b,
                                  const double* z, double* res, double* part, double* colsq, double scale,
                                  double tol, int32_t nonfinite_stop, int32_t record, double* errs, int64_t errs_cap,
                                  int64_t k, Control* ctl, cudaStream_t st) {
  k_res_rows<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(A, lda, m, n, x, b, z, ctl, res);
  const int nchunks = (m + kResChunk - 1) / kResChunk;
  k_res_cols<<<dim3((unsigned)((n + 255) / 256), (unsigned)nchunks), 256, 0, st>>>(A, lda, m, n, res, ctl, part);
  k_res_norm<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, nchunks, part, ctl, colsq);
  k_res_decide<<<1, 1024, 0, st>>>(n, colsq, scale, tol, nonfinite_stop, record, errs, errs_cap, k, ctl);
  return cudaGetLastError();
}

size_t residual_check_part_len(int m, int n) { return (size_t)((m + kResChunk - 1) / kResChunk) * n; }
}  // namespace rebk

// rebk_shard.cu — per-rank REBK pieces for the row-sharded multi-GPU path
// (BASELINE config 3).
//
// A is row-sharded: rank p holds, for every row block I_b, the local rows
// q of I_b with floor(q * P / |I_b|) == p (interleaved, so every row block is
// spread over all ranks and the row step is balanced).  z and b follow the
// rows; x is replicated.  One iteration (step_rebk, solvers.py:324-337) is
//   u_p  = A_p[:, J]ᵀ z_p            (rebk_shard_colstep)     -> allreduce(u)
//   z_p -= s_J A_p[:, J] u            (rebk_shard_zupdate)
//   r_p  = A_p[I_p, :] x - b + z      (rebk_shard_rowstep)
//   dx_p = A_p[I_p, :]ᵀ r_p                                      -> allreduce(dx)
//   x   -= s_I dx                     (rebk_shard_xupdate)
// The two allreduces (|J| and n doubles) run between these calls on the
// caller's communicator (NCCL through torch.distributed).  Every reduction
// here is fixed-order (two-pass), so a rank's results are reproducible.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rebk_internal.h"

namespace rebk {

constexpr int kShardThreads = 256;
constexpr int kShardRowsPerCta = 256;  // colstep: z rows per partial
constexpr int kTransRows = 32;         // rowstep: local rows of I per partial of Aᵀ r

// pass 1: part[cta][j] = Σ_{r in this CTA's rows} A[r, c_lo + j] z[r].
// Warp w takes rows w, w + 8, ...; lane l accumulates columns l, l + 32, ...
// (up to kColPerLane of them), so every row is one coalesced sweep with all of
// its loads in flight; the 8 warp sums are then added in warp order.
constexpr int kColPerLane = 16;  // |J| <= 512
__global__ void __launch_bounds__(kShardThreads) shard_colstep_part(const double* __restrict__ A, int64_t lda,
                                                                  int64_t m, int64_t c_lo, int nJ,
                                                                  const double* __restrict__ z,
                                                                  double* __restrict__ part) {
  __shared__ double s_acc[kShardThreads / 32][kColPerLane * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kShardRowsPerCta;
  const int64_t r1 = r0 + kShardRowsPerCta < m ? r0 + kShardRowsPerCta : m;
  double acc[kColPerLane];
#pragma unroll
  for (int t = 0; t < kColPerLane; ++t) acc[t] = 0.0;
  constexpr int W = kShardThreads / 32;
  int64_t r = r0 + warp;
  for (; r + 3 * W < r1; r += 4 * W) {  // four rows per step: 4 x kColPerLane loads in flight per lane
    double zz[4];
    double v[4][kColPerLane];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      zz[u] = __ldg(z + r + u * W);
      const double* au = A + (r + u * W) * lda + c_lo;
#pragma unroll
      for (int t = 0; t < kColPerLane; ++t) {
        const int j = lane + 32 * t;
        v[u][t] = j < nJ ? __ldg(au + j) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int t = 0; t < kColPerLane; ++t) acc[t] = fma(v[u][t], zz[u], acc[t]);
  }
  for (; r + W < r1; r += 2 * W) {  // two rows per step
    const double z0 = __ldg(z + r), z1 = __ldg(z + r + W);
    const double* a0 = A + r * lda + c_lo;
    const double* a1 = a0 + W * lda;
    double v0[kColPerLane], v1[kColPerLane];
#pragma unroll
    for (int t = 0; t < kColPerLane; ++t) {
      const int j = lane + 32 * t;
      v0[t] = j < nJ ? __ldg(a0 + j) : 0.0;
      v1[t] = j < nJ ? __ldg(a1 + j) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < kColPerLane; ++t) {
      acc[t] = fma(v0[t], z0, acc[t]);
      acc[t] = fma(v1[t], z1, acc[t]);
    }
  }
  if (r < r1) {
    const double zr = __ldg(z + r);
    const double* a = A + r * lda + c_lo;
#pragma unroll
    for (int t = 0; t < kColPerLane; ++t) {
      const int j = lane + 32 * t;
      if (j < nJ) acc[t] = fma(__ldg(a + j), zr, acc[t]);
    }
  }
#pragma unroll
  for (int t = 0; t < kColPerLane; ++t) s_acc[warp][lane + 32 * t] = acc[t];
  __syncthreads();
  for (int j = threadIdx.x; j < nJ; j += kShardThreads) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kShardThreads / 32; ++w) v += s_acc[w][j];
    part[(int64_t)blockIdx.x * nJ + j] = v;
  }
}
// pass 2: out[j] = Σ_q part[q][j]: a CTA per 32 entries, warp w sums parts
// w, w + 8, ... (loads in flight across the warp's iterations), then the 8
// warp sums in order
__global__ void __launch_bounds__(256) shard_sum_parts(const double* __restrict__ part, int nparts, int len,
                                                       double* __restrict__ out) {
  __shared__ double s_w[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (j < len) {
#pragma unroll 4
    for (int q = warp; q < nparts; q += 8) acc += part[(int64_t)q * len + j];
  }
  s_w[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && j < len) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += s_w[w][lane];
    out[j] = v;
  }
}
// z[r] -= s * Σ_j A[r, c_lo + j] u[j]  (one warp per row)
__global__ void __launch_bounds__(kShardThreads) shard_zupdate(const double* __restrict__ A, int64_t lda, int64_t m,
                                                              int64_t c_lo, int nJ, double s,
                                                              const double* __restrict__ u, double* __restrict__ z) {
  __shared__ double su[kColPerLane * 32];
  const int lane = threadIdx.x & 31;
  const bool fits = nJ <= kColPerLane * 32;
  if (fits)
    for (int j = threadIdx.x; j < nJ; j += kShardThreads) su[j] = u[j];
  __syncthreads();
  const int64_t r = ((int64_t)blockIdx.x * kShardThreads + threadIdx.x) >> 5;
  if (r >= m) return;
  const double* a = A + r * lda + c_lo;
  double acc = 0.0;
  if (fits) {
    // the row's loads all in flight, then the FMAs in the lane's column order
    double v[kColPerLane];
#pragma unroll
    for (int t = 0; t < kColPerLane; ++t) {
      const int j = lane + 32 * t;
      v[t] = j < nJ ? __ldg(a + j) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < kColPerLane; ++t) {
      const int j = lane + 32 * t;
      if (j < nJ) acc = fma(v[t], su[j], acc);
    }
  } else {
    for (int j = lane; j < nJ; j += 32) acc = fma(__ldg(a + j), u[j], acc);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) z[r] = z[r] - s * acc;
}

// r[q] = (A[rows_q, :] x - b[rows_q]) + z[rows_q]: one CTA per local row,
// thread-strided dot, fixed-order block reduction
__global__ void __launch_bounds__(kShardThreads) shard_rowresid(const double* __restrict__ A, int64_t lda, int64_t n,
                                                              const int64_t* __restrict__ rows, int64_t nrows,
                                                              const double* __restrict__ x,
                                                              const double* __restrict__ b,
                                                              const double* __restrict__ z, double* __restrict__ r) {
  __shared__ double s_w[kShardThreads / 32];
  const int64_t q = blockIdx.x;
  if (q >= nrows) return;
  const int64_t row = rows[q];
  const double* a = A + row * lda;
  double s0 = 0.0, s1 = 0.0;
  int64_t c = threadIdx.x;
  for (; c + kShardThreads < n; c += 2 * kShardThreads) {
    s0 = fma(__ldg(a + c), __ldg(x + c), s0);
    s1 = fma(__ldg(a + c + kShardThreads), __ldg(x + c + kShardThreads), s1);
  }
  if (c < n) s0 = fma(__ldg(a + c), __ldg(x + c), s0);
  double acc = s0 + s1;
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < kShardThreads / 32; ++w) v += s_w[w];
    v -= b[row];
    if (z) v += z[row];
    r[q] = v;
  }
}

// part[p][c] = Σ_{q in chunk p} A[rows_q, c] r[q]  (thread per column, kTransRows rows per chunk)
__global__ void shard_rowtrans_part(const double* __restrict__ A, int64_t lda, int64_t n,
                                    const int64_t* __restrict__ rows, int64_t nrows, const double* __restrict__ r,
                                    double* __restrict__ part) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t q0 = (int64_t)blockIdx.y * kTransRows;
  const int64_t q1 = q0 + kTransRows < nrows ? q0 + kTransRows : nrows;
  double acc = 0.0;
  for (int64_t q = q0; q < q1; ++q) acc = fma(__ldg(A + rows[q] * lda + c), r[q], acc);
  part[(int64_t)blockIdx.y * n + c] = acc;
}

__global__ void shard_xupdate(int64_t n, double s, const double* __restrict__ dx, double* __restrict__ x) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) x[c] = x[c] - s * dx[c];
}

// Σ (x - x*)^2, one CTA, fixed order
__global__ void shard_err2(int64_t n, const double* __restrict__ x, const double* __restrict__ xs, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
    const double d = x[c] - xs[c];
    acc = fma(d, d, acc);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    *out = s;
  }
}

cudaError_t shard_colstep(const double* A, int64_t lda, int64_t m, int64_t c_lo, int nJ, const double* z, double* u,
                          double* scratch, cudaStream_t st) {
  const int nparts = (int)((m + kShardRowsPerCta - 1) / kShardRowsPerCta);
  shard_colstep_part<<<nparts, kShardThreads, 0, st>>>(A, lda, m, c_lo, nJ, z, scratch);
  shard_sum_parts<<<(nJ + 31) / 32, 256, 0, st>>>(scratch, nparts, nJ, u);
  return cudaGetLastError();
}

cudaError_t shard_zupd(const double* A, int64_t lda, int64_t m, int64_t c_lo, int nJ, double s, const double* u,
                       double* z, cudaStream_t st) {
  const int64_t warps = m;
  shard_zupdate<<<(unsigned)((warps * 32 + kShardThreads - 1) / kShardThreads), kShardThreads, 0, st>>>(A, lda, m, c_lo,
                                                                                                        nJ, s, u, z);
  return cudaGetLastError();
}

cudaError_t shard_rowstep(const double* A, int64_t lda, int64_t n, const int64_t* rows, int64_t nrows, const double* x,
                          const double* b, const double* z, double* r_scratch, double* dx, cudaStream_t st) {
  if (nrows <= 0) return cudaMemsetAsync(dx, 0, n * sizeof(double), st);
  shard_rowresid<<<(unsigned)nrows, kShardThreads, 0, st>>>(A, lda, n, rows, nrows, x, b, z, r_scratch);
  const int nparts = (int)((nrows + kTransRows - 1) / kTransRows);
  double* part = r_scratch + nrows;
  shard_rowtrans_part<<<dim3((unsigned)((n + 255) / 256), (unsigned)nparts), 256, 0, st>>>(A, lda, n, rows, nrows,
                                                                                         r_scratch, part);
  shard_sum_parts<<<(unsigned)((n + 31) / 32), 256, 0, st>>>(part, nparts, (int)n, dx);
  return cudaGetLastError();
}

size_t shard_colstep_scratch(int64_t m, int64_t nJ) {
  return (size_t)((m + kShardRowsPerCta - 1) / kShardRowsPerCta) * (size_t)nJ;
}
size_t shard_rowstep_scratch(int64_t nrows, int64_t n) {
  return (size_t)nrows + (size_t)((nrows + kTransRows - 1) / kTransRows) * (size_t)n + 1;
}

cudaError_t shard_xupd(int64_t n, double s, const double* dx, double* x, cudaStream_t st) {
  shard_xupdate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, s, dx, x);
  return cudaGetLastError();
}

cudaError_t shard_err(int64_t n, const double* x, const double* xs, double* out, cudaStream_t st) {
  shard_err2<<<1, 1024, 0, st>>>(n, x, xs, out);
  return cudaGetLastError();
}

}  // namespace rebk

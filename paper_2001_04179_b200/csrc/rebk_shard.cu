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
constexpr int kShardRowsPerCta = 64;

// pass 1: part[cta][j] = Σ_{r in this CTA's rows} A[r, c_lo + j] z[r]
__global__ void shard_colstep_part(const double* __restrict__ A, int64_t lda, int64_t m, int64_t c_lo, int nJ,
                                   const double* __restrict__ z, double* __restrict__ part) {
  const int64_t r0 = (int64_t)blockIdx.x * kShardRowsPerCta;
  const int64_t r1 = r0 + kShardRowsPerCta < m ? r0 + kShardRowsPerCta : m;
  for (int j = threadIdx.x; j < nJ; j += kShardThreads) {
    double acc = 0.0;
    for (int64_t r = r0; r < r1; ++r) acc = fma(__ldg(A + r * lda + c_lo + j), z[r], acc);
    part[(int64_t)blockIdx.x * nJ + j] = acc;
  }
}

// pass 2: u[j] = Σ_cta part[cta][j]
__global__ void shard_sum_parts(const double* __restrict__ part, int nparts, int len, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= len) return;
  double acc = 0.0;
  for (int q = 0; q < nparts; ++q) acc += part[(int64_t)q * len + j];
  out[j] = acc;
}

// z[r] -= s * Σ_j A[r, c_lo + j] u[j]  (one warp per row)
__global__ void shard_zupdate(const double* __restrict__ A, int64_t lda, int64_t m, int64_t c_lo, int nJ, double s,
                              const double* __restrict__ u, double* __restrict__ z) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * kShardThreads + threadIdx.x) >> 5;
  if (r >= m) return;
  double acc = 0.0;
  for (int j = lane; j < nJ; j += 32) acc = fma(__ldg(A + r * lda + c_lo + j), u[j], acc);
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) z[r] = z[r] - s * acc;
}

// r[q] = (A[rows_q, :] x - b[rows_q]) + z[rows_q]  (one warp per local row)
__global__ void shard_rowresid(const double* __restrict__ A, int64_t lda, int64_t n, const int64_t* __restrict__ rows,
                               int64_t nrows, const double* __restrict__ x, const double* __restrict__ b,
                               const double* __restrict__ z, double* __restrict__ r) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * kShardThreads + threadIdx.x) >> 5;
  if (q >= nrows) return;
  const int64_t row = rows[q];
  double acc = 0.0;
  for (int64_t c = lane; c < n; c += 32) acc = fma(__ldg(A + row * lda + c), x[c], acc);
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    double v = acc - b[row];
    if (z) v += z[row];
    r[q] = v;
  }
}

// dx[c] = Σ_q A[rows_q, c] r[q]  (thread per column, rows in order)
__global__ void shard_rowtrans(const double* __restrict__ A, int64_t lda, int64_t n, const int64_t* __restrict__ rows,
                               int64_t nrows, const double* __restrict__ r, double* __restrict__ dx) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double acc = 0.0;
  for (int64_t q = 0; q < nrows; ++q) acc = fma(__ldg(A + rows[q] * lda + c), r[q], acc);
  dx[c] = acc;
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
  shard_sum_parts<<<(nJ + 127) / 128, 128, 0, st>>>(scratch, nparts, nJ, u);
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
  if (nrows > 0)
    shard_rowresid<<<(unsigned)((nrows * 32 + kShardThreads - 1) / kShardThreads), kShardThreads, 0, st>>>(
        A, lda, n, rows, nrows, x, b, z, r_scratch);
  shard_rowtrans<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A, lda, n, rows, nrows, r_scratch, dx);
  return cudaGetLastError();
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

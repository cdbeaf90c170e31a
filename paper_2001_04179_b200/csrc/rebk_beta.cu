// rebk_beta.cu — block spectral norms on the device:
// sigma_1(B)^2 for every block B of a dense partition, the numerator of the
// reference's beta = max_b sigma_1(B_b)^2 / ||B_b||_F^2 (rates.py:76-90,
// used by solvers.py:180-185 and the CLI's x-suffixed stepsizes,
// cli.py:288-302).  The reference takes a one-sided Jacobi SVD of every
// materialised block (factorizations.py); here every block runs Lanczos
// with full reorthogonalisation on its small Gram operator
//   axis 0 (row block,    tau x n): M = B Bᵀ,  v -> B (Bᵀ v)
//   axis 1 (column block, m x tau): M = Bᵀ B,  v -> Bᵀ (B v)
// so A is streamed twice per Lanczos step and never materialised or
// squared: all blocks of the partition advance together (one pass over A per
// product), which makes each step HBM-bound.  The top Ritz value of the
// Lanczos tridiagonal T_k (warp-parallel Sturm multisection) converges to
// sigma_1^2 from below at the Kaniel-Paige rate; a block stops when the Ritz
// value is stable to 1e-15 for three consecutive steps, when the Krylov space
// is exhausted (k = tau) or on breakdown.  Every reduction has a fixed order,
// so the result is deterministic.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "rebk_internal.h"

namespace rebk {

namespace beta {

constexpr int kT = 256;
constexpr int kRowChunk = 512;  // axis 1: rows of A per partial of Bᵀ t
constexpr int kColChunk = 2048;  // axis 0: columns of A per partial of B t

struct Blocks {
  const int64_t* ptr;  // [nb+1] block bounds along the axis
  const int64_t* voff;  // [nb] offset of the block's Lanczos basis (kmax+1 vectors of tau)
  const int64_t* woff;  // [nb] offset of the block's entries in one partial slice (sum of tau)
  int64_t wtot;         // entries per partial slice
  int nb, kmax;
  int32_t* done;        // [nb] 1 = converged / exhausted
};

// v0: deterministic, positive pseudo-random entries (never orthogonal to the
// top eigenvector of a Gram matrix with a positive Perron vector, and
// generic otherwise), normalised
__global__ void k_init(Blocks bl, double* V, double* alpha, double* betas, double* theta, int32_t* stable) {
  const int b = blockIdx.x;
  const int64_t tau = bl.ptr[b + 1] - bl.ptr[b];
  double* v = V + bl.voff[b];
  __shared__ double red[kT];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < tau; e += kT) {
    uint64_t h = (uint64_t)(e + 1) * 0x9E3779B97F4A7C15ull ^ (uint64_t)(b + 7) * 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
    h *= 0x94D049BB133111EBull;
    h ^= h >> 29;
    const double x = 0.5 + (double)(h >> 11) * 0x1.0p-53;
    v[e] = x;
    s += x * x;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double inv = 1.0 / sqrt(red[0]);
  for (int64_t e = threadIdx.x; e < tau; e += kT) v[e] *= inv;
  if (threadIdx.x == 0) {
    bl.done[b] = 0;
    theta[b] = 0.0;
    stable[b] = 0;
  }
  (void)alpha;
  (void)betas;
}

// ---- product 1: t = Bᵀ v (axis 0, length n) or B v (axis 1, length m) ----
// axis 0: one thread per column, v in shared memory, rows in order
__global__ void __launch_bounds__(kT) k_t_rows(const double* __restrict__ A, int64_t lda, int64_t n, Blocks bl,
                                               const double* __restrict__ V, int k, double* __restrict__ T) {
  extern __shared__ double sv[];
  const int b = blockIdx.y;
  if (bl.done[b]) return;
  const int64_t p0 = bl.ptr[b], tau = bl.ptr[b + 1] - p0;
  const double* v = V + bl.voff[b] + (int64_t)k * tau;
  for (int64_t i = threadIdx.x; i < tau; i += kT) sv[i] = v[i];
  __syncthreads();
  const int64_t col = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (col >= n) return;
  const double* a = A + p0 * lda + col;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t i = 0;
  for (; i + 4 <= tau; i += 4) {
    s0 += a[(i + 0) * lda] * sv[i + 0];
    s1 += a[(i + 1) * lda] * sv[i + 1];
    s2 += a[(i + 2) * lda] * sv[i + 2];
    s3 += a[(i + 3) * lda] * sv[i + 3];
  }
  for (; i < tau; ++i) s0 += a[i * lda] * sv[i];
  T[(int64_t)b * n + col] = (s0 + s1) + (s2 + s3);
}

// axis 1: one warp per row of A, lanes across the block's tau columns
__global__ void __launch_bounds__(kT) k_t_cols(const double* __restrict__ A, int64_t lda, int64_t m, Blocks bl,
                                               const double* __restrict__ V, int k, double* __restrict__ T) {
  extern __shared__ double sv[];
  const int b = blockIdx.y;
  if (bl.done[b]) return;
  const int64_t p0 = bl.ptr[b], tau = bl.ptr[b + 1] - p0;
  const double* v = V + bl.voff[b] + (int64_t)k * tau;
  for (int64_t i = threadIdx.x; i < tau; i += kT) sv[i] = v[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RPB = 32;  // rows per CTA
  for (int rr = warp; rr < RPB; rr += kT / 32) {
    const int64_t r = (int64_t)blockIdx.x * RPB + rr;
    if (r >= m) break;
    const double* a = A + r * lda + p0;
    double s = 0.0;
    for (int64_t j = lane; j < tau; j += 32) s += a[j] * sv[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) T[(int64_t)b * m + r] = s;
  }
}

// ---- product 2: w = B t (axis 0) or Bᵀ t (axis 1), as partial slices ----
// axis 0: slice s covers columns [s*kColChunk, ...): warp per row of the block
__global__ void __launch_bounds__(kT) k_w_rows(const double* __restrict__ A, int64_t lda, int64_t n, Blocks bl,
                                               const double* __restrict__ T, double* __restrict__ W) {
  __shared__ double st[kColChunk];
  const int b = blockIdx.y, s = blockIdx.x;
  if (bl.done[b]) return;
  const int64_t p0 = bl.ptr[b], tau = bl.ptr[b + 1] - p0;
  const int64_t c0 = (int64_t)s * kColChunk, c1 = min(n, c0 + (int64_t)kColChunk);
  for (int64_t c = c0 + threadIdx.x; c < c1; c += kT) st[c - c0] = T[(int64_t)b * n + c];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t i = warp; i < tau; i += kT / 32) {
    const double* a = A + (p0 + i) * lda;
    double acc = 0.0;
    for (int64_t c = c0 + lane; c < c1; c += 32) acc += a[c] * st[c - c0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) W[(int64_t)s * bl.wtot + bl.woff[b] + i] = acc;
  }
}

// axis 1: slice s covers rows [s*kRowChunk, ...): thread per block column
__global__ void __launch_bounds__(kT) k_w_cols(const double* __restrict__ A, int64_t lda, int64_t m, Blocks bl,
                                               const double* __restrict__ T, double* __restrict__ W) {
  __shared__ double st[kRowChunk];
  const int b = blockIdx.y, s = blockIdx.x;
  if (bl.done[b]) return;
  const int64_t p0 = bl.ptr[b], tau = bl.ptr[b + 1] - p0;
  const int64_t r0 = (int64_t)s * kRowChunk, r1 = min(m, r0 + (int64_t)kRowChunk);
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kT) st[r - r0] = T[(int64_t)b * m + r];
  __syncthreads();
  for (int64_t j = threadIdx.x; j < tau; j += kT) {
    const double* a = A + r0 * lda + p0 + j;
    double s0 = 0.0, s1 = 0.0;
    int64_t r = r0;
    for (; r + 2 <= r1; r += 2) {
      s0 += a[(r - r0) * lda] * st[r - r0];
      s1 += a[(r - r0 + 1) * lda] * st[r - r0 + 1];
    }
    if (r < r1) s0 += a[(r - r0) * lda] * st[r - r0];
    W[(int64_t)s * bl.wtot + bl.woff[b] + j] = s0 + s1;
  }
}

// ---- Lanczos step k of every live block (one CTA per block) -------------
// fixed-order block reduction of one value per thread
__device__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = kT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// number of eigenvalues of the symmetric tridiagonal (a, b) below x (Sturm)
__device__ int sturm_below(const double* a, const double* b, int n, double x) {
  int cnt = 0;
  double q = a[0] - x;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < n; ++i) {
    const double qq = (q == 0.0) ? 1e-300 : q;
    q = a[i] - x - b[i - 1] * b[i - 1] / qq;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// largest eigenvalue of the n x n tridiagonal: warp 0, 33-section of a
// Gershgorin bracket until it stops shrinking
__device__ double top_ritz(const double* a, const double* b, int n) {
  const int lane = threadIdx.x & 31;
  double lo = a[0] - (n > 1 ? fabs(b[0]) : 0.0), hi = a[0] + (n > 1 ? fabs(b[0]) : 0.0);
  for (int i = 1; i < n; ++i) {
    const double r = fabs(b[i - 1]) + (i + 1 < n ? fabs(b[i]) : 0.0);
    lo = fmin(lo, a[i] - r);
    hi = fmax(hi, a[i] + r);
  }
  for (int round = 0; round < 64; ++round) {
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    // all n eigenvalues below x <=> x is above the top one
    const unsigned above = __ballot_sync(0xffffffffu, sturm_below(a, b, n, x) == n);
    double nlo = lo, nhi = hi;
    if (above) {
      const int l = __ffs(above) - 1;
      nhi = __shfl_sync(0xffffffffu, x, l);
      if (l > 0) nlo = __shfl_sync(0xffffffffu, x, l - 1);
    } else {
      nlo = __shfl_sync(0xffffffffu, x, 31);
    }
    if (!(nhi - nlo < hi - lo)) break;
    lo = nlo;
    hi = nhi;
  }
  return 0.5 * (lo + hi);
}

__global__ void __launch_bounds__(kT) k_step(Blocks bl, int nslices, const double* __restrict__ W, double* V, int k,
                                             double* alpha, double* betas, double* theta, int32_t* stable,
                                             int32_t* steps, double* wbuf) {
  __shared__ double red[kT];
  __shared__ double h[1024];
  const int b = blockIdx.x;
  if (bl.done[b]) return;
  const int64_t tau = bl.ptr[b + 1] - bl.ptr[b];
  double* Vb = V + bl.voff[b];
  double* w = wbuf + bl.woff[b];
  const double* vk = Vb + (int64_t)k * tau;
  // w = Σ_s W[s] (slice order), alpha_k = w . v_k
  double part = 0.0;
  for (int64_t e = threadIdx.x; e < tau; e += kT) {
    double s = 0.0;
    for (int q = 0; q < nslices; ++q) s += W[(int64_t)q * bl.wtot + bl.woff[b] + e];
    w[e] = s;
    part += s * vk[e];
  }
  const double ak = block_sum(part, red);
  const double bprev = k > 0 ? betas[(int64_t)b * bl.kmax + k - 1] : 0.0;
  for (int64_t e = threadIdx.x; e < tau; e += kT) {
    double x = w[e] - ak * vk[e];
    if (k > 0) x -= bprev * Vb[(int64_t)(k - 1) * tau + e];
    w[e] = x;
  }
  __syncthreads();
  // full reorthogonalisation against v_0..v_k, two classical Gram-Schmidt passes
  for (int pass = 0; pass < 2; ++pass) {
    for (int i0 = 0; i0 <= k; i0 += 1024) {
      const int i1 = min(k + 1, i0 + 1024);
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int i = i0 + warp; i < i1; i += kT / 32) {
        const double* vi = Vb + (int64_t)i * tau;
        double s = 0.0;
        for (int64_t e = lane; e < tau; e += 32) s += w[e] * vi[e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) h[i - i0] = s;
      }
      __syncthreads();
      for (int64_t e = threadIdx.x; e < tau; e += kT) {
        double x = w[e];
        for (int i = i0; i < i1; ++i) x -= h[i - i0] * Vb[(int64_t)i * tau + e];
        w[e] = x;
      }
      __syncthreads();
    }
  }
  double nn = 0.0;
  for (int64_t e = threadIdx.x; e < tau; e += kT) nn += w[e] * w[e];
  const double bk = sqrt(block_sum(nn, red));
  if (threadIdx.x == 0) {
    alpha[(int64_t)b * bl.kmax + k] = ak;
    betas[(int64_t)b * bl.kmax + k] = bk;
  }
  const bool breakdown = !(bk > 1e-14 * fabs(ak)) || k + 1 >= tau || k + 1 >= bl.kmax;
  if (!breakdown) {
    double* vn = Vb + (int64_t)(k + 1) * tau;
    const double inv = 1.0 / bk;
    for (int64_t e = threadIdx.x; e < tau; e += kT) vn[e] = w[e] * inv;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const double th = top_ritz(alpha + (int64_t)b * bl.kmax, betas + (int64_t)b * bl.kmax, k + 1);
    if (threadIdx.x == 0) {
      const double prev = theta[b];
      int st = (fabs(th - prev) <= 1e-15 * fabs(th)) ? stable[b] + 1 : 0;
      theta[b] = th;
      stable[b] = st;
      steps[b] = k + 1;
      if (breakdown || st >= 3) bl.done[b] = 1;
    }
  }
}

}  // namespace beta

// sigma_1^2 of every block of a contiguous partition of the dense A (device),
// written to theta_out[nb] (host); steps_out[nb] = Lanczos steps taken
cudaError_t block_sigma1_sq(const double* A, int64_t lda, int64_t m, int64_t n, int axis, int64_t nb,
                            const int64_t* h_ptr, int kmax_req, double* theta_out, int32_t* steps_out,
                            cudaStream_t stream) {
  using namespace beta;
  int64_t tau_max = 0, wtot = 0;
  std::vector<int64_t> voff(nb), woff(nb);
  int kmax = std::max(1, kmax_req);
  for (int64_t b = 0; b < nb; ++b) tau_max = std::max(tau_max, h_ptr[b + 1] - h_ptr[b]);
  kmax = (int)std::min<int64_t>(kmax, tau_max);
  int64_t vtot = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t tau = h_ptr[b + 1] - h_ptr[b];
    voff[b] = vtot;
    vtot += (int64_t)(std::min<int64_t>(kmax, tau) + 1) * tau;
    woff[b] = wtot;
    wtot += tau;
  }
  const int64_t q = axis == 0 ? n : m;
  const int nslices = (int)(axis == 0 ? (n + kColChunk - 1) / kColChunk : (m + kRowChunk - 1) / kRowChunk);
  std::vector<void*> ptrs;
  cudaError_t e = cudaSuccess;
  auto alloc = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMallocAsync(p, std::max<size_t>(bytes, 8), stream);
    if (e == cudaSuccess) ptrs.push_back(*p);
  };
  int64_t *d_ptr = nullptr, *d_voff = nullptr, *d_woff = nullptr;
  int32_t *d_done = nullptr, *d_stable = nullptr, *d_steps = nullptr;
  double *d_V = nullptr, *d_T = nullptr, *d_W = nullptr, *d_w = nullptr, *d_alpha = nullptr, *d_beta = nullptr,
         *d_theta = nullptr;
  alloc((void**)&d_ptr, (nb + 1) * 8);
  alloc((void**)&d_voff, nb * 8);
  alloc((void**)&d_woff, nb * 8);
  alloc((void**)&d_done, nb * 4);
  alloc((void**)&d_stable, nb * 4);
  alloc((void**)&d_steps, nb * 4);
  alloc((void**)&d_V, vtot * 8);
  alloc((void**)&d_T, (size_t)nb * q * 8);
  alloc((void**)&d_W, (size_t)nslices * wtot * 8);
  alloc((void**)&d_w, wtot * 8);
  alloc((void**)&d_alpha, (size_t)nb * kmax * 8);
  alloc((void**)&d_beta, (size_t)nb * kmax * 8);
  alloc((void**)&d_theta, nb * 8);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_ptr, h_ptr, (nb + 1) * 8, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_voff, voff.data(), nb * 8, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_woff, woff.data(), nb * 8, cudaMemcpyHostToDevice, stream);
  Blocks bl{d_ptr, d_voff, d_woff, wtot, (int)nb, kmax, d_done};
  const size_t sv_bytes = (size_t)tau_max * 8;
  if (e == cudaSuccess && sv_bytes > 48 * 1024) {
    e = cudaFuncSetAttribute(k_t_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sv_bytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_t_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sv_bytes);
  }
  if (e == cudaSuccess) {
    k_init<<<(unsigned)nb, kT, 0, stream>>>(bl, d_V, d_alpha, d_beta, d_theta, d_stable);
    e = cudaGetLastError();
  }
  std::vector<int32_t> hdone(nb);
  for (int k = 0; k < kmax && e == cudaSuccess; ++k) {
    if (axis == 0) {
      k_t_rows<<<dim3((unsigned)((n + kT - 1) / kT), (unsigned)nb), kT, sv_bytes, stream>>>(A, lda, n, bl, d_V, k,
                                                                                          d_T);
      k_w_rows<<<dim3((unsigned)nslices, (unsigned)nb), kT, 0, stream>>>(A, lda, n, bl, d_T, d_W);
    } else {
      k_t_cols<<<dim3((unsigned)((m + 31) / 32), (unsigned)nb), kT, sv_bytes, stream>>>(A, lda, m, bl, d_V, k,
                                                                                      d_T);
      k_w_cols<<<dim3((unsigned)nslices, (unsigned)nb), kT, 0, stream>>>(A, lda, m, bl, d_T, d_W);
    }
    k_step<<<(unsigned)nb, kT, 0, stream>>>(bl, nslices, d_W, d_V, k, d_alpha, d_beta, d_theta, d_stable, d_steps,
                                            d_w);
    e = cudaGetLastError();
    if (e == cudaSuccess && (k % 8 == 7 || k + 1 == kmax)) {
      e = cudaMemcpyAsync(hdone.data(), d_done, nb * 4, cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
      if (e == cudaSuccess && std::all_of(hdone.begin(), hdone.end(), [](int32_t v) { return v != 0; })) break;
    }
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(theta_out, d_theta, nb * 8, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess && steps_out) e = cudaMemcpyAsync(steps_out, d_steps, nb * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  for (void* p : ptrs) cudaFreeAsync(p, stream);
  cudaStreamSynchronize(stream);
  return e;
}

}  // namespace rebk

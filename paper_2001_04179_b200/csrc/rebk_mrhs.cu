// rebk_mrhs.cu — multi-right-hand-side fp32 REBK (BASELINE config 5).
//
// All RHS share one block sequence (the sequence never depends on b,
// solvers.py:8-12), so with X (n x R), Z (m x R), B (m x R) the four block
// products of step_rebk (solvers.py:283-295) become GEMMs:
//   U  = A_Jᵀ Z                 (|J| x R)
//   Z -= s_J A_J U
//   Rr = A_I X - B_I + Z_I      (|I| x R)
//   X -= s_I A_Iᵀ Rr
// Round 1 runs them through cuBLAS FP32 GEMMs (optionally the BF16x9 FP32
// emulation on tensor cores; single-pass TF32 misses the 1e-4 tolerance,
// SURVEY hard part 6), split-K for the two reductions, captured as one CUDA graph per chunk
// of 64 iterations (the block sequence of a chunk is sampled on the device
// first; the host only needs it to address the GEMMs).  The per-column stopping rule (each RHS records the first check
// with ||X_c - X*_c|| <= tol_c; the run ends when every column has crossed)
// runs on the device; the final state is the one at that iteration, obtained
// by restoring the chunk's checkpoint and replaying (the sequence and the
// GEMMs are deterministic).
//
// cuBLAS is opened with dlopen at first use (librebk.so has no link-time
// cuBLAS dependency).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/rebk.h"
#include "rebk_internal.h"
#include <stdio.h>
#include <stdlib.h>

namespace rebk {

// ---- minimal dlopen'ed cuBLAS ------------------------------------------------
typedef void* cublasHandle_t;
enum { CUBLAS_OP_N = 0, CUBLAS_OP_T = 1 };
enum { CUBLAS_DEFAULT_MATH = 0, CUBLAS_PEDANTIC_MATH = 2, CUBLAS_FP32_EMULATED_BF16X9_MATH = 4 };

struct CublasApi {
  bool ok = false;
  int (*create)(cublasHandle_t*) = nullptr;
  int (*destroy)(cublasHandle_t) = nullptr;
  int (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
  int (*set_math)(cublasHandle_t, int) = nullptr;
  int (*set_workspace)(cublasHandle_t, void*, size_t) = nullptr;
  int (*sgemm)(cublasHandle_t, int, int, int, int, int, const float*, const float*, int, const float*, int,
               const float*, float*, int) = nullptr;
  int (*sgemm_sb)(cublasHandle_t, int, int, int, int, int, const float*, const float*, int, long long, const float*,
                  int, long long, const float*, float*, int, long long, int) = nullptr;
};

static CublasApi& cublas() {
  static CublasApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* names[] = {"/usr/local/cuda/lib64/libcublas.so.12", "libcublas.so.12", "libcublas.so"};
  void* h = nullptr;
  for (const char* nm : names) {
    h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
    if (h) break;
  }
  if (!h) return api;
  api.create = (int (*)(cublasHandle_t*))dlsym(h, "cublasCreate_v2");
  api.destroy = (int (*)(cublasHandle_t))dlsym(h, "cublasDestroy_v2");
  api.set_stream = (int (*)(cublasHandle_t, cudaStream_t))dlsym(h, "cublasSetStream_v2");
  api.set_math = (int (*)(cublasHandle_t, int))dlsym(h, "cublasSetMathMode");
  api.set_workspace = (int (*)(cublasHandle_t, void*, size_t))dlsym(h, "cublasSetWorkspace_v2");
  api.sgemm = (int (*)(cublasHandle_t, int, int, int, int, int, const float*, const float*, int, const float*, int,
                       const float*, float*, int))dlsym(h, "cublasSgemm_v2");
  api.sgemm_sb = (int (*)(cublasHandle_t, int, int, int, int, int, const float*, const float*, int, long long,
                          const float*, int, long long, const float*, float*, int, long long, int))
      dlsym(h, "cublasSgemmStridedBatched");
  api.ok = api.create && api.destroy && api.set_stream && api.set_math && api.set_workspace && api.sgemm &&
           api.sgemm_sb;
  return api;
}

// ---- small kernels -------------------------------------------------------------
// Rr = Z_I - B_I, or -B_I without a column sweep (pointers already offset to row r_lo)
__global__ void mrhs_init_r(const float* __restrict__ ZI, const float* __restrict__ BI, float* __restrict__ Rr,
                            int64_t count) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) Rr[t] = (ZI ? ZI[t] : 0.0f) - BI[t];
}

// out[e] = init[e] + Σ_{b<nb} part[b][e]  (fixed order: split-K reduction)
__global__ void mrhs_reduce_parts(const float* __restrict__ part, int nb, int64_t len, const float* __restrict__ init,
                                  float* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= len) return;
  float acc = init ? init[e] : 0.0f;
#pragma unroll 8
  for (int b = 0; b < nb; ++b) acc += part[(int64_t)b * len + e];
  out[e] = acc;
}

// per-column ||X_c - X*_c||^2, two deterministic stages: partial sums over
// row chunks of 256 rows (grid: column groups of 32 x row chunks), then one
// thread per column sums the chunks in order and does the crossing logic.
constexpr int kCheckRows = 256;
__global__ void mrhs_check_part(const float* __restrict__ X, const float* __restrict__ Xs, int64_t n, int R,
                                double* __restrict__ part) {
  __shared__ double sp[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int w = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.y * kCheckRows;
  const int64_t r1 = r0 + kCheckRows < n ? r0 + kCheckRows : n;
  double acc = 0.0;
  if (c < R)
    for (int64_t i = r0 + w; i < r1; i += 8) {
      const double d = (double)X[i * R + c] - (double)Xs[i * R + c];
      acc = fma(d, d, acc);
    }
  sp[w][threadIdx.x & 31] = acc;
  __syncthreads();
  if (w == 0 && c < R) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += sp[q][threadIdx.x & 31];
    part[(int64_t)blockIdx.y * R + c] = s;
  }
}

__global__ void mrhs_check_final(const double* __restrict__ part, int nchunks, int R, const double* __restrict__ tol,
                                 int64_t k, int64_t* iters, double* errs, double* errs_at, int32_t* n_done) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= R) return;
  double s = 0.0;
  for (int q = 0; q < nchunks; ++q) s += part[(int64_t)q * R + c];
  const double e = sqrt(s);
  errs[c] = e;
  if (iters[c] < 0 && e <= tol[c]) {
    iters[c] = k;
    errs_at[c] = e;
    atomicAdd(n_done, 1);
  }
}

// ---- host orchestration --------------------------------------------------------

#define MR_TRY(expr)                                                   \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) {                                           \
      snprintf(errbuf, errlen, "%s: %s", #expr, cudaGetErrorString(_e)); \
      return -2;                                                       \
    }                                                                  \
  } while (0)
#define MB_TRY(expr)                                                   \
  do {                                                                 \
    int _s = (expr);                                                   \
    if (_s != 0) {                                                     \
      snprintf(errbuf, errlen, "%s: cuBLAS status %d", #expr, _s);     \
      return -2;                                                       \
    }                                                                  \
  } while (0)

// Default FP32 (SIMT) GEMMs: measured faster end to end than the BF16x9
// emulation here (the emulation adds an inf/NaN scan and patch kernels per
// GEMM, profiles/r01_c5_launches.txt).  REBK_MRHS_MATH=bf16x9 selects it.
static int mrhs_math_mode() {
  const char* s = getenv("REBK_MRHS_MATH");
  if (s && !strcmp(s, "bf16x9")) return CUBLAS_FP32_EMULATED_BF16X9_MATH;
  if (s && !strcmp(s, "default")) return CUBLAS_DEFAULT_MATH;  // "pedantic" (or anything else): FP32
  return CUBLAS_PEDANTIC_MATH;
}

int run_mrhs(const MrhsRun& w, const SampleParams& sp_template, const SampleParams* unused, int64_t* iters_out,
             double* errs_out, double* loop_ms, int64_t* k_final, char* errbuf, size_t errlen, cudaStream_t stream,
             int* math_used) {
  (void)unused;
  // default: the hand-written tcgen05 3xTF32 kernels (rebk_mrhs_tc.cu);
  // REBK_MRHS_MATH=pedantic|default|bf16x9 selects the cuBLAS path
  const char* mm = getenv("REBK_MRHS_MATH");
  if (w.At && (!mm || !strcmp(mm, "tc"))) {
    int nJm = 1, nIm = 1;
    for (int64_t b = 0; b < w.cfg->n_row_blocks; ++b)
      nIm = std::max<int>(nIm, (int)(w.cfg->row_ptr[b + 1] - w.cfg->row_ptr[b]));
    if (w.extended)
      for (int64_t b = 0; b < w.cfg->n_col_blocks; ++b)
        nJm = std::max<int>(nJm, (int)(w.cfg->col_ptr[b + 1] - w.cfg->col_ptr[b]));
    if (mrhs_tc_supported(w.m, w.n, w.R, nJm, nIm)) {
      const int r = run_mrhs_tc(w, sp_template, iters_out, errs_out, loop_ms, k_final, errbuf, errlen, stream);
      if (r != -3) {  // -3: partition not supported by the tensor-core path
        *math_used = 6;
        return r;
      }
    }
  }
  CublasApi& cb = cublas();
  if (!cb.ok) {
    snprintf(errbuf, errlen, "cuBLAS could not be loaded (dlopen libcublas.so.12)");
    return -2;
  }
  const rebk_cfg* cfg = w.cfg;
  const int R = w.R;
  const int64_t m = w.m, n = w.n, lda = w.lda;
  const bool checking = cfg->stop_mode == 0;
  cublasHandle_t h = nullptr;
  MB_TRY(cb.create(&h));
  struct HGuard {
    CublasApi& cb;
    cublasHandle_t h;
    ~HGuard() { cb.destroy(h); }
  } hg{cb, h};
  MB_TRY(cb.set_stream(h, stream));
  const int math = mrhs_math_mode();
  if (cb.set_math(h, math) != 0) MB_TRY(cb.set_math(h, CUBLAS_DEFAULT_MATH));
  *math_used = math;
  void* ws = nullptr;
  const size_t ws_bytes = 64u << 20;
  MR_TRY(cudaMallocAsync(&ws, ws_bytes, stream));
  MB_TRY(cb.set_workspace(h, ws, ws_bytes));

  int nJmax = 1, nImax = 1;
  for (int64_t b = 0; b < cfg->n_row_blocks; ++b) nImax = std::max<int>(nImax, (int)(cfg->row_ptr[b + 1] - cfg->row_ptr[b]));
  if (w.extended)
    for (int64_t b = 0; b < cfg->n_col_blocks; ++b)
      nJmax = std::max<int>(nJmax, (int)(cfg->col_ptr[b + 1] - cfg->col_ptr[b]));
  float *U, *Rr, *Xsnap = nullptr, *Zsnap = nullptr;
  double *d_tol, *d_errs, *d_errs_at;
  int64_t* d_iters;
  int32_t* d_ndone;
  Plan* d_plan;
  const int64_t CH = 64;
  MR_TRY(cudaMallocAsync((void**)&U, sizeof(float) * nJmax * R, stream));
  MR_TRY(cudaMallocAsync((void**)&Rr, sizeof(float) * nImax * R, stream));
  MR_TRY(cudaMallocAsync((void**)&Xsnap, sizeof(float) * n * R, stream));
  if (w.extended) MR_TRY(cudaMallocAsync((void**)&Zsnap, sizeof(float) * m * R, stream));
  MR_TRY(cudaMallocAsync((void**)&d_tol, sizeof(double) * R, stream));
  MR_TRY(cudaMallocAsync((void**)&d_errs, sizeof(double) * R, stream));
  MR_TRY(cudaMallocAsync((void**)&d_errs_at, sizeof(double) * R, stream));
  MR_TRY(cudaMallocAsync((void**)&d_iters, sizeof(int64_t) * R, stream));
  MR_TRY(cudaMallocAsync((void**)&d_ndone, sizeof(int32_t), stream));
  MR_TRY(cudaMallocAsync((void**)&d_plan, sizeof(Plan) * CH, stream));
  const int nchk = (int)((n + kCheckRows - 1) / kCheckRows);
  double* d_cpart;
  MR_TRY(cudaMallocAsync((void**)&d_cpart, sizeof(double) * nchk * R, stream));
  auto launch_check = [&](int64_t k) -> cudaError_t {
    mrhs_check_part<<<dim3((R + 31) / 32, nchk), 256, 0, stream>>>(w.X, w.Xs, n, R, d_cpart);
    mrhs_check_final<<<(R + 127) / 128, 128, 0, stream>>>(d_cpart, nchk, R, d_tol, k, d_iters, d_errs, d_errs_at,
                                                           d_ndone);
    return cudaGetLastError();
  };
  // split-K: the two reductions (over m for U, over n for Rr) have tiny
  // outputs (R x |J|, R x |I|), so one GEMM would occupy a handful of SMs;
  // batch them over K chunks and sum the partials in a fixed order.
  const int64_t kc_m = 2048, kc_n = 512;
  // full K chunks (possibly none: a dimension shorter than one chunk is all remainder)
  const int64_t nb_m = m / kc_m, nb_n = n / kc_n;
  float* P;
  const int64_t plen = std::max<int64_t>((int64_t)nJmax * R * (nb_m + 1), (int64_t)nImax * R * (nb_n + 1));
  MR_TRY(cudaMallocAsync((void**)&P, sizeof(float) * plen, stream));
  std::vector<double> tol(R);
  for (int c = 0; c < R; ++c) tol[c] = w.tols ? w.tols[c] : cfg->tol;
  MR_TRY(cudaMemcpyAsync(d_tol, tol.data(), sizeof(double) * R, cudaMemcpyHostToDevice, stream));
  MR_TRY(cudaMemsetAsync(d_iters, 0xff, sizeof(int64_t) * R, stream));  // -1
  MR_TRY(cudaMemsetAsync(d_ndone, 0, sizeof(int32_t), stream));
  MR_TRY(cudaMemsetAsync(d_errs_at, 0, sizeof(double) * R, stream));

  auto enqueue_iter = [&](const Plan& pl, int64_t k, bool do_check) -> int {
    const int nJ = pl.c_hi - pl.c_lo, nI = pl.r_hi - pl.r_lo;
    const float one = 1.0f, zero = 0.0f;
    if (w.extended) {
      const float mcs = (float)(-pl.c_scale);
      // U = Σ_chunks Z_chunkᵀ-rows x A_J chunk (split over m), then the z update
      const int64_t ulen = (int64_t)nJ * R;
      if (nb_m > 0)
        MB_TRY(cb.sgemm_sb(h, CUBLAS_OP_N, CUBLAS_OP_T, R, nJ, (int)kc_m, &one, w.Z, R, kc_m * R, w.A + pl.c_lo,
                           (int)lda, kc_m * lda, &zero, P, R, ulen, (int)nb_m));
      const int64_t rem = m - nb_m * kc_m;
      if (rem > 0)
        MB_TRY(cb.sgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, R, nJ, (int)rem, &one, w.Z + nb_m * kc_m * R, R,
                        w.A + pl.c_lo + nb_m * kc_m * lda, (int)lda, &zero, P + nb_m * ulen, R));
      mrhs_reduce_parts<<<(unsigned)((ulen + 255) / 256), 256, 0, stream>>>(P, (int)(nb_m + (rem > 0)), ulen, nullptr,
                                                                            U);
      MR_TRY(cudaGetLastError());
      MB_TRY(cb.sgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, R, (int)m, nJ, &mcs, U, R, w.A + pl.c_lo, (int)lda, &one, w.Z, R));
    }
    const int64_t cnt = (int64_t)nI * R;
    mrhs_init_r<<<(unsigned)((cnt + 255) / 256), 256, 0, stream>>>(w.extended ? w.Z + (int64_t)pl.r_lo * R : nullptr,
                                                                  w.B + (int64_t)pl.r_lo * R, Rr, cnt);
    MR_TRY(cudaGetLastError());
    const float* AI = w.A + (int64_t)pl.r_lo * lda;
    const float mrs = (float)(-pl.r_scale);
    {
      // Rr += Σ_chunks X_chunk x A_I chunk (split over n)
      if (nb_n > 0)
        MB_TRY(cb.sgemm_sb(h, CUBLAS_OP_N, CUBLAS_OP_N, R, nI, (int)kc_n, &one, w.X, R, kc_n * R, AI, (int)lda, kc_n,
                           &zero, P, R, cnt, (int)nb_n));
      const int64_t rem = n - nb_n * kc_n;
      if (rem > 0)
        MB_TRY(cb.sgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, R, nI, (int)rem, &one, w.X + nb_n * kc_n * R, R,
                        AI + nb_n * kc_n, (int)lda, &zero, P + nb_n * cnt, R));
      mrhs_reduce_parts<<<(unsigned)((cnt + 255) / 256), 256, 0, stream>>>(P, (int)(nb_n + (rem > 0)), cnt, Rr, Rr);
      MR_TRY(cudaGetLastError());
    }
    MB_TRY(cb.sgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, R, (int)n, nI, &mrs, Rr, R, AI, (int)lda, &one, w.X, R));
    if (do_check) MR_TRY(launch_check(k));
    return 0;
  };

  cudaEvent_t ev0, ev1;
  MR_TRY(cudaEventCreate(&ev0));
  MR_TRY(cudaEventCreate(&ev1));
  MR_TRY(cudaEventRecord(ev0, stream));
  int64_t K = cfg->max_iters;
  bool all_done = false;
  if (checking) {
    MR_TRY(launch_check(0));
    int32_t nd = 0;
    MR_TRY(cudaMemcpyAsync(&nd, d_ndone, sizeof nd, cudaMemcpyDeviceToHost, stream));
    MR_TRY(cudaStreamSynchronize(stream));
    if (nd == R) {
      all_done = true;
      K = 0;
    }
  }
  std::vector<Plan> hplan(CH);
  SampleParams sp = sp_template;
  for (int64_t k0 = 1; !all_done && k0 <= cfg->max_iters; k0 += CH) {
    const int64_t cnt = std::min(CH, cfg->max_iters - k0 + 1);
    MR_TRY(launch_sample_plan(sp, k0, cnt, d_plan, nullptr, stream));
    MR_TRY(cudaMemcpyAsync(hplan.data(), d_plan, sizeof(Plan) * cnt, cudaMemcpyDeviceToHost, stream));
    MR_TRY(cudaStreamSynchronize(stream));
    if (checking) {
      MR_TRY(cudaMemcpyAsync(Xsnap, w.X, sizeof(float) * n * R, cudaMemcpyDeviceToDevice, stream));
      if (w.extended) MR_TRY(cudaMemcpyAsync(Zsnap, w.Z, sizeof(float) * m * R, cudaMemcpyDeviceToDevice, stream));
    }
    // one CUDA graph per chunk: the ~8 launches of an iteration cost more
    // host time than the GPU spends on them
    const bool use_graph = !getenv("REBK_MRHS_NO_GRAPH");
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    if (use_graph) MR_TRY(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    for (int64_t q = 0; q < cnt; ++q) {
      const int64_t k = k0 + q;
      int rc = enqueue_iter(hplan[q], k, checking && (k % cfg->check_stride == 0 || k == cfg->max_iters));
      if (rc) {
        if (use_graph) {
          cudaStreamEndCapture(stream, &graph);
          if (graph) cudaGraphDestroy(graph);
        }
        return rc;
      }
    }
    if (use_graph) {
      MR_TRY(cudaStreamEndCapture(stream, &graph));
      MR_TRY(cudaGraphInstantiate(&gexec, graph, 0));
      MR_TRY(cudaGraphLaunch(gexec, stream));
      MR_TRY(cudaStreamSynchronize(stream));
      cudaGraphExecDestroy(gexec);
      cudaGraphDestroy(graph);
    }
    if (checking) {
      int32_t nd = 0;
      MR_TRY(cudaMemcpyAsync(&nd, d_ndone, sizeof nd, cudaMemcpyDeviceToHost, stream));
      MR_TRY(cudaStreamSynchronize(stream));
      if (nd == R) {
        std::vector<int64_t> it(R);
        MR_TRY(cudaMemcpy(it.data(), d_iters, sizeof(int64_t) * R, cudaMemcpyDeviceToHost));
        K = *std::max_element(it.begin(), it.end());
        all_done = true;
        if (K < k0 + cnt - 1) {  // rewind to the chunk start and replay up to K exactly
          MR_TRY(cudaMemcpyAsync(w.X, Xsnap, sizeof(float) * n * R, cudaMemcpyDeviceToDevice, stream));
          if (w.extended) MR_TRY(cudaMemcpyAsync(w.Z, Zsnap, sizeof(float) * m * R, cudaMemcpyDeviceToDevice, stream));
          for (int64_t k = k0; k <= K; ++k) {
            int rc = enqueue_iter(hplan[k - k0], k, false);
            if (rc) return rc;
          }
        }
      }
    }
  }
  MR_TRY(cudaEventRecord(ev1, stream));
  MR_TRY(cudaStreamSynchronize(stream));
  float ms = 0.f;
  MR_TRY(cudaEventElapsedTime(&ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  *loop_ms = ms;
  *k_final = K;
  if (iters_out) MR_TRY(cudaMemcpy(iters_out, d_iters, sizeof(int64_t) * R, cudaMemcpyDeviceToHost));
  if (errs_out) MR_TRY(cudaMemcpy(errs_out, d_errs_at, sizeof(double) * R, cudaMemcpyDeviceToHost));
  cudaFreeAsync(U, stream);
  cudaFreeAsync(Rr, stream);
  cudaFreeAsync(Xsnap, stream);
  if (Zsnap) cudaFreeAsync(Zsnap, stream);
  cudaFreeAsync(d_tol, stream);
  cudaFreeAsync(d_errs, stream);
  cudaFreeAsync(d_errs_at, stream);
  cudaFreeAsync(d_iters, stream);
  cudaFreeAsync(d_ndone, stream);
  cudaFreeAsync(d_plan, stream);
  cudaFreeAsync(P, stream);
  cudaFreeAsync(d_cpart, stream);
  cudaFreeAsync(ws, stream);
  cudaStreamSynchronize(stream);
  return 0;
}

}  // namespace rebk

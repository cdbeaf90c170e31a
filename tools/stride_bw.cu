// HBM read bandwidth of C3's column-block access pattern versus a contiguous
// stream: each of 148 CTAs reads its rows of a 200000 x 10000 fp64 matrix,
// 500 columns (4000 B) per row at an 80 KB row stride, with plain 16-byte
// loads (no TMA) -- against the same number of bytes read contiguously.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stride_bw tools/stride_bw.cu && tools/stride_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_strided(const double* __restrict__ A, long m, long lda, int c0, int w,
                                                 double* out) {
  double acc = 0.0;
  const long r0 = m * blockIdx.x / gridDim.x, r1 = m * (blockIdx.x + 1) / gridDim.x;
  const int w2 = w / 2;
  for (long e = threadIdx.x; e < (r1 - r0) * w2; e += blockDim.x) {
    const long r = r0 + e / w2;
    const int c = c0 + 2 * (int)(e % w2);
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(A + r * lda + c));
    acc += v.x + v.y;
  }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void __launch_bounds__(512) k_contig(const double* __restrict__ A, long n, double* out) {
  double acc = 0.0;
  for (long i = 2 * ((long)blockIdx.x * blockDim.x + threadIdx.x); i < n; i += 2L * gridDim.x * blockDim.x) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(A + i));
    acc += v.x + v.y;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const long m = 200000, lda = 10000;
  double *A, *out;
  cudaMalloc(&A, m * lda * sizeof(double));
  cudaMemset(A, 0, m * lda * sizeof(double));
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_it = [&](auto launch) {
    launch();
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return best;
  };
  const double bytes = (double)m * 500 * 8;
  for (int cta_per_sm : {1, 2, 4}) {
    float ms = time_it([&] { k_strided<<<sms * cta_per_sm, 512>>>(A, m, lda, 500 * 7, 500, out); });
    printf("{\"pattern\": \"column block 500 of 10000 (4000 B per 80 KB row)\", \"ctas\": %d, \"gbs\": %.1f}\n",
           sms * cta_per_sm, bytes / (ms * 1e-3) / 1e9);
  }
  for (int cta_per_sm : {1, 4}) {
    float ms = time_it([&] { k_contig<<<sms * cta_per_sm, 512>>>(A + 7L * m * 500, m * 500, out); });
    printf("{\"pattern\": \"contiguous 800 MB\", \"ctas\": %d, \"gbs\": %.1f}\n", sms * cta_per_sm,
           bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}

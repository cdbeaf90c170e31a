// hbm_sustained.cu — pure-read HBM bandwidth of a 4 GB buffer by launch length: the C3 solve streams for ~160 ms under
// the board's power cap, the 7.3 TB/s of tools/l2_bw.cu is a 1.6 ms launch.  Same loads as l2_bw.cu (ld.global.cg.v4.f64,
// grid-stride over the whole buffer), reps = 3 ... 400 passes per launch, CUDA events around each launch; also a strided
// variant that reads the buffer as C3's column block is read (each CTA its own contiguous slice, 4 KB pieces).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_sustained tools/hbm_sustained.cu && tools/hbm_sustained
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_read(const double4* __restrict__ p, size_t n4, int reps, double* out) {
  double acc = 0.0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      double4 v;
      asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + i));
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.678) out[0] = acc;
}
// each CTA streams its own contiguous 1/G of the buffer (the ownership pattern of the C3 kernel's row slices)
__global__ void __launch_bounds__(512) k_read_own(const double4* __restrict__ p, size_t n4, int reps, double* out) {
  double acc = 0.0;
  const size_t lo = n4 * blockIdx.x / gridDim.x, hi = n4 * (blockIdx.x + 1) / gridDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      double4 v;
      asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + i));
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 4096ull << 20;
  double *buf, *out;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  cudaMalloc(&out, 8);
  const size_t n4 = bytes / 32;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int own = 0; own < 2; ++own)
    for (int reps : {3, 12, 50, 100, 200, 400}) {
      float ms = 0;
      for (int t = 0; t < 2; ++t) {
        cudaEventRecord(e0);
        if (own) k_read_own<<<sms * 4, 512>>>((const double4*)buf, n4, reps, out);
        else k_read<<<sms * 4, 512>>>((const double4*)buf, n4, reps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("%s, %3d passes over 4 GB: %7.1f ms, %7.1f GB/s\n", own ? "per-CTA contiguous slices" : "grid-stride sweep          ", reps, ms,
             (double)bytes * reps / (ms * 1e-3) / 1e9);
    }
  return 0;
}

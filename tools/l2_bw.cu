// L2 and HBM read bandwidth on this B200 (C1's A = 8 MB is
// L2-resident, so its roofline is the L2's, measured here).  Each CTA reads
// its slice of a buffer with 16-byte loads (ld.global.cg: no L1 reuse),
// sums it (so the loads are not dead), repeated `reps` times in one launch;
// CUDA events around the launch.  Buffers of 8-64 MB stay in the 126 MB L2
// after the first pass; 4 GB streams from HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bw tools/l2_bw.cu && tools/l2_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_read(const double4* __restrict__ p, size_t n4, int reps, double* out) {
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      double4 v;
      asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                   : "l"(p + i));
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t sizes_mb[] = {8, 16, 32, 64, 96, 4096};
  double* out;
  cudaMalloc(&out, 8);
  printf("{\"sm_count\": %d, \"points\": [", sms);
  for (int s = 0; s < 6; ++s) {
    const size_t bytes = sizes_mb[s] << 20;
    double* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    const size_t n4 = bytes / 32;
    const int reps = bytes > (1ull << 30) ? 3 : (int)(8192ull / sizes_mb[s]);
    k_read<<<sms * 4, 512>>>((const double4*)buf, n4, 1, out);  // warm (and fill L2)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
      cudaEventRecord(e0);
      k_read<<<sms * 4, 512>>>((const double4*)buf, n4, reps, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%s{\"buffer_mb\": %zu, \"reps\": %d, \"read_gbs\": %.1f}", s ? ", " : "", sizes_mb[s], reps,
           (double)bytes * reps / (best * 1e-3) / 1e9);
    cudaFree(buf);
  }
  printf("]}\n");
  return 0;
}

// own_bw.cu — does the OWNERSHIP of rows matter for HBM read bandwidth on C3's column-block pattern?
// A = 200000 x 10000 fp64 (16 GB); the column block is 500 columns (4000 B) per row at an 80 KB pitch (800 MB).
// Modes: 0 each CTA owns a contiguous range of rows (the C3 kernel's split), 1 chunks of `ch` rows dealt round-robin
// to the CTAs (at any moment the chip reads one neighbourhood of rows).  Plain 16-byte loads, G CTAs of 512 threads,
// `reps` passes per launch (sustained, ~100 ms).  Also the same two ownerships on a CONTIGUOUS 800 MB slab (pitch 4000 B).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/own_bw tools/own_bw.cu && tools/own_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_own(const double* __restrict__ A, long m, long pitch, int w, int mode, int ch, int reps,
                                             double* out) {
  double acc = 0.0;
  const int G = gridDim.x, g = blockIdx.x;
  const int w2 = w / 2;
  for (int rep = 0; rep < reps; ++rep) {
    if (mode == 0) {
      const long r0 = m * g / G, r1 = m * (g + 1) / G;
      for (long e = threadIdx.x; e < (r1 - r0) * w2; e += blockDim.x) {
        const long r = r0 + e / w2;
        const int c = 2 * (int)(e % w2);
        double2 v;
        asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(A + r * pitch + c));
        acc += v.x + v.y;
      }
    } else {
      const long nchunk = (m + ch - 1) / ch;
      for (long cidx = g; cidx < nchunk; cidx += G) {
        const long r0 = cidx * ch, r1 = r0 + ch < m ? r0 + ch : m;
        for (long e = threadIdx.x; e < (r1 - r0) * w2; e += blockDim.x) {
          const long r = r0 + e / w2;
          const int c = 2 * (int)(e % w2);
          double2 v;
          asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(A + r * pitch + c));
          acc += v.x + v.y;
        }
      }
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const long m = 200000;
  double *A, *out;
  cudaMalloc(&A, m * 10000 * sizeof(double));
  cudaMemset(A, 0, m * 10000 * sizeof(double));
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)m * 500 * 8;
  for (long pitch : {10000L, 500L})
    for (int cps : {1, 4})
      for (int mode = 0; mode < 2; ++mode)
        for (int ch : {47, 8}) {
          if (mode == 0 && ch != 47) continue;
          const int reps = 800;
          float ms = 0;
          for (int t = 0; t < 2; ++t) {
            cudaEventRecord(e0);
            k_own<<<sms * cps, 512>>>(A, m, pitch, 500, mode, ch, reps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
          }
          printf("pitch %5ld doubles, %d CTA/SM, %s: %7.1f ms, %7.1f GB/s\n", pitch, cps,
                 mode == 0 ? "contiguous row range per CTA   " : (ch == 47 ? "47-row chunks dealt round-robin" : " 8-row chunks dealt round-robin"),
                 ms, bytes * reps / (ms * 1e-3) / 1e9);
        }
  return 0;
}

// tma_own_bw.cu — the C3 kernel's column pass as a pure TMA stream (no consumers): 148 CTAs, a ring of NS stages,
// boxes of 250 columns x 47 rows (94 KB) of a 200000 x 10000 fp64 matrix, two boxes per 47-row chunk (the 500-column
// block).  Ownership 0: CTA g streams its contiguous range of rows (the kernel's split); 1: the 47-row chunks are
// dealt round-robin to the CTAs (the chip sweeps one neighbourhood of rows at a time).  `reps` passes per launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tools/tma_own_bw.cu -o tools/tma_own_bw
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"

using namespace rebk;

constexpr int BW = 250, BH = 47;

__global__ void __launch_bounds__(128, 1)
    k_stream(const __grid_constant__ CUtensorMap map, int m, int own, int ns, int reps, int c_lo) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[8];
  const int G = gridDim.x, g = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    const uint32_t bytes = BW * BH * 8;
    const long nchunk = (m + BH - 1) / BH;
    const long r0 = (long)m * g / G, r1 = (long)m * (g + 1) / G;
    const long mine = own ? (nchunk - g + G - 1) / G : (r1 - r0 + BH - 1) / BH;
    const long nbox = 2 * mine * reps;
    long issued = 0, done = 0;
    uint32_t ph = 0;
    auto issue = [&](long i) {
      const long ci = (i / 2) % mine;
      const int half = (int)(i & 1);
      const long row = own ? (ci * G + g) * BH : r0 + ci * BH;
      const int s = (int)(i % ns);
      mbar_arrive_expect_tx(&bar[s], bytes);  // rows past the owner's range are simply read too (same bytes per box)
      tma_load_2d(smem + (size_t)s * ((bytes + 127) & ~127u), &map, c_lo + half * BW, (int)row, &bar[s]);
    };
    for (; issued < ns && issued < nbox; ++issued) issue(issued);
    while (done < nbox) {
      const int s = (int)(done % ns);
      mbar_wait(&bar[s], (ph >> s) & 1u);
      ph ^= 1u << s;
      ++done;
      if (issued < nbox) issue(issued++);
    }
  }
  __syncthreads();
}

int main() {
  const int m = 200000, n = 10000;
  double* A;
  cudaMalloc(&A, (size_t)m * n * 8);
  cudaMemset(A, 0, (size_t)m * n * 8);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)f;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
  cuuint64_t strides[1] = {(cuuint64_t)n * 8};
  cuuint32_t box[2] = {BW, BH}, es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 600;
  for (int ns : {2, 4})
    for (int own = 0; own < 2; ++own) {
      float ms = 0;
      for (int t = 0; t < 2; ++t) {
        cudaEventRecord(e0);
        k_stream<<<148, 128, (size_t)ns * 94208 + 1024>>>(map, m, own, ns, reps, 3000);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaEventElapsedTime(&ms, e0, e1);
      }
      // bytes actually requested: boxes x 94,000 B
      const long nchunk = (m + BH - 1) / BH;
      double boxes = 0;
      for (int g = 0; g < 148; ++g) {
        const long r0 = (long)m * g / 148, r1 = (long)m * (g + 1) / 148;
        boxes += 2.0 * (own ? (nchunk - g + 147) / 148 : (r1 - r0 + BH - 1) / BH);
      }
      printf("ring of %d x 94 KB, %s: %7.1f ms for %d passes, %7.1f GB/s (%.1f us per 800 MB pass)\n", ns,
             own ? "47-row chunks dealt round-robin" : "contiguous row range per CTA   ", ms, reps,
             boxes * BW * BH * 8 * reps / (ms * 1e-3) / 1e9, 1e3 * ms / reps);
    }
  return 0;
}

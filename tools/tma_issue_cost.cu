// tma_issue_cost.cu — how long does the ISSUING thread spend on one TMA
// instruction?  clock64 around back-to-back issues (no waits in between):
//   a) 8 tensor loads (16 KB boxes, 8 barriers) from one thread
//   b) 8 L2 tensor prefetches from one thread
//   c) 8 L2 tensor prefetches, one per lane, in ONE warp instruction
//   d) 32 prefetches, one per lane, in one instruction
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tools/tma_issue_cost.cu -o tools/tma_issue_cost
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"

using namespace rebk;

__global__ void __launch_bounds__(128, 1) k_cost(const __grid_constant__ CUtensorMap map, int ncols, int nrows, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int boxes_x = ncols / 32, boxes_y = nrows / 128;
  auto box = [&](int i, int& c0, int& c1) {
    const int b = (blockIdx.x * 131 + i * 7) % (boxes_x * boxes_y);
    c0 = (b % boxes_x) * 32;
    c1 = (b / boxes_x) * 128;
  };
  long long t[6] = {0, 0, 0, 0, 0, 0};
  for (int rep = 0; rep < 4; ++rep) {
    if (tid == 0) {
      long long t0 = clock64();
      for (int i = 0; i < 8; ++i) {
        int c0, c1;
        box(rep * 100 + i, c0, c1);
        mbar_arrive_expect_tx(&bar[i], 16384);
        tma_load_2d(smem + i * 16384, &map, c0, c1, &bar[i]);
      }
      long long t1 = clock64();
      for (int i = 0; i < 8; ++i) mbar_wait(&bar[i], rep & 1);
      long long t2 = clock64();
      for (int i = 0; i < 8; ++i) {
        int c0, c1;
        box(rep * 100 + 50 + i, c0, c1);
        tma_prefetch_l2_2d(&map, c0, c1);
      }
      long long t3 = clock64();
      if (rep == 3) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; }
    }
    __syncthreads();
    if (tid < 32) {
      long long t0 = clock64();
      if (tid < 8) {
        int c0, c1;
        box(rep * 100 + 60 + tid, c0, c1);
        tma_prefetch_l2_2d(&map, c0, c1);
      }
      __syncwarp();
      long long t1 = clock64();
      {
        int c0, c1;
        box(rep * 100 + 70 + tid, c0, c1);
        tma_prefetch_l2_2d(&map, c0, c1);
      }
      __syncwarp();
      long long t2 = clock64();
      if (rep == 3 && tid == 0) { t[3] = t1 - t0; t[4] = t2 - t1; }
    }
    __syncthreads();
  }
  if (tid == 0) for (int i = 0; i < 5; ++i) out[blockIdx.x * 8 + i] = t[i];
}

int main() {
  const int nrows = 4096, ncols = 2048;  // 32 MB, L2-resident after the first touch
  float* d;
  cudaMalloc(&d, (size_t)nrows * ncols * 4);
  cudaMemset(d, 0, (size_t)nrows * ncols * 4);
  long long* dout;
  cudaMalloc(&dout, 148 * 8 * 8);
  cudaFuncSetAttribute(k_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 1024);
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)f;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)ncols, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {(cuuint64_t)ncols * 4};
  cuuint32_t es[2] = {1, 1};
  cuuint32_t box[2] = {32, 128};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int pass = 0; pass < 2; ++pass) {
    k_cost<<<148, 128, 8 * 16384 + 1024>>>(map, ncols, nrows, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
  }
  std::vector<long long> h(148 * 8);
  cudaMemcpy(h.data(), dout, h.size() * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"issue 8 tensor loads back to back (one thread)", "then wait for all 8 to land",
                         "issue 8 L2 tensor prefetches back to back (one thread)", "8 prefetches, one per lane, ONE instruction",
                         "32 prefetches, one per lane, ONE instruction"};
  for (int i = 0; i < 5; ++i) {
    std::vector<long long> v;
    for (int b = 0; b < 148; ++b) v.push_back(h[b * 8 + i]);
    std::sort(v.begin(), v.end());
    printf("%-58s median %6lld cycles (min %lld, max %lld)\n", names[i], v[74], v[0], v[147]);
  }
  return 0;
}

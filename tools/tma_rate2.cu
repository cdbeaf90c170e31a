// tma_rate2.cu — what limits ONE issuing thread to ~640 cycles per TMA box
// (tools/tma_rate.cu)?  Same L2-resident fp32 matrix, one CTA per SM, no
// consumers; box 32 floats x 128 rows (SW128, 16 KB).  Variants:
//   0  lane 0 of warp 0, NS stages, wait oldest -> reissue (the baseline)
//   1  lanes 0 and 1 of warp 0, each with its own NS stages (same warp)
//   2  lane 0 of warps 0 and 1 (different warps)
//   3  lane 0 of warp 0, batched: wait for the two oldest stages, then issue two boxes back to back
//   4  lane 0 of warp 0, a stage = two boxes (16 KB + 8 KB) on ONE barrier (the C5 kernel's stage)
//   5  as 4, lane 0 of warps 0 and 1 alternating stages
//   6  as 0 but the wait is mbarrier.try_wait with a suspend-time hint
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tools/tma_rate2.cu -o tools/tma_rate2
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"

using namespace rebk;

constexpr int kBars = 32;
constexpr uint32_t kBoxA = 32 * 128 * 4, kBoxB = 32 * 64 * 4;

__global__ void __launch_bounds__(384, 1)
    k_rate(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int ncols, int nrows,
           int ns, int nstage, int variant, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kBars];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kBars; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int boxes_x = ncols / 32, boxes_y = nrows / 128;
  const long long t0 = clock64();
  int pidx = -1, nprod = 1;
  if (variant == 1) { nprod = 2; if (warp == 0 && lane < 2) pidx = lane; }
  else if (variant == 2 || variant == 5) { nprod = 2; if (lane == 0 && warp < 2) pidx = warp; }
  else if (tid == 0) pidx = 0;
  const bool two_box = variant == 4 || variant == 5;
  const uint32_t stage_bytes = two_box ? kBoxA + kBoxB : kBoxA;
  if (pidx >= 0) {
    const int mine = nstage / nprod;
    auto issue = [&](int i) {  // i: this producer's i-th stage
      const int gi = i * nprod + pidx;
      const int b = (blockIdx.x * 131 + gi * 7) % (boxes_x * boxes_y);
      const int s = pidx * ns + i % ns;
      unsigned char* dst = smem + (size_t)s * stage_bytes;
      mbar_arrive_expect_tx(&bar[s], stage_bytes);
      tma_load_2d(dst, &mapA, (b % boxes_x) * 32, (b / boxes_x) * 128, &bar[s]);
      if (two_box) tma_load_2d(dst + kBoxA, &mapB, (b % boxes_x) * 32, (b / boxes_x) * 128, &bar[s]);
    };
    auto wait = [&](int i, uint32_t& ph) {
      const int s = pidx * ns + i % ns;
      if (variant == 6) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
              : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"((ph >> (i % ns)) & 1u), "r"(2000u) : "memory");
      } else {
        mbar_wait(&bar[s], (ph >> (i % ns)) & 1u);
      }
      ph ^= 1u << (i % ns);
    };
    uint32_t ph = 0;
    int issued = 0, done = 0;
    for (; issued < ns && issued < mine; ++issued) issue(issued);
    if (variant == 3) {
      while (done < mine) {
        wait(done, ph); ++done;
        if (done < mine) { wait(done, ph); ++done; }
        if (issued < mine) { issue(issued); ++issued; }
        if (issued < mine) { issue(issued); ++issued; }
      }
    } else {
      while (done < mine) {
        wait(done, ph);
        ++done;
        if (issued < mine) { issue(issued); ++issued; }
      }
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  const int nrows = 1024, ncols = 2048;
  float* d;
  cudaMalloc(&d, (size_t)nrows * ncols * 4);
  cudaMemset(d, 0, (size_t)nrows * ncols * 4);
  long long* dcyc;
  cudaMalloc(&dcyc, 148 * 8);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)f;
  CUtensorMap mapA, mapB;
  cuuint64_t dims[2] = {(cuuint64_t)ncols, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {(cuuint64_t)ncols * 4};
  cuuint32_t es[2] = {1, 1};
  cuuint32_t boxA[2] = {32, 128}, boxB[2] = {32, 64};
  enc(&mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mapB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const char* names[] = {"1 thread, wait oldest -> reissue", "lanes 0,1 of ONE warp", "lane 0 of TWO warps",
                         "1 thread, waits 2 then issues 2 back to back", "1 thread, stage = 2 boxes (16+8 KB) on one barrier",
                         "2 warps alternating 2-box stages", "1 thread, try_wait with suspend hint"};
  for (int variant = 0; variant < 7; ++variant)
    for (int ns : {2, 4}) {
      const int nstage = 2000;
      const bool two_box = variant == 4 || variant == 5;
      const size_t sb = two_box ? kBoxA + kBoxB : kBoxA;
      const int nprod = (variant == 1 || variant == 2 || variant == 5) ? 2 : 1;
      k_rate<<<148, 384, (size_t)ns * nprod * sb + 1024>>>(mapA, mapB, ncols, nrows, ns, nstage, variant, dcyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<long long> h(148);
      cudaMemcpy(h.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.end());
      printf("variant %d (%-50s) %d stages in flight per producer: %6.1f B/clk/SM, %5.0f cycles per stage (%zu KB)\n", variant,
             names[variant], ns, (double)nstage * sb / h[74], (double)h[74] / nstage, sb / 1024);
    }
  return 0;
}

// tma_rate.cu — per-SM ingest rate of TMA 2D loads from an L2-resident fp32
// matrix, by box shape and number of boxes in flight: one CTA per SM, thread 0
// keeps NS boxes in flight through a ring of mbarriers and reissues each as it
// lands (no consumers).  Also: the same bytes by plain 16-byte loads of all
// threads, and both at once (TMA for 2/3 of the bytes, loads for 1/3).
// Question (C5 kernel): is a stage stream of 128-byte-row boxes bound by the
// TMA unit's request rate rather than by L2?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tools/tma_rate.cu -o tools/tma_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"

using namespace rebk;

constexpr int kMaxStages = 8;

// mode 0: TMA only; 1: plain loads only; 2: both (the loads fetch half as many bytes as the TMA boxes)
__global__ void __launch_bounds__(384, 1)
    k_tma_rate(const __grid_constant__ CUtensorMap map, const float* __restrict__ base, int box_w, int box_h, int ncols,
               int nrows, int ns, int nbox, int mode, int nprod, long long* cycles, float* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[4 * kMaxStages];
  const int tid = threadIdx.x;
  const uint32_t box_bytes = (uint32_t)box_w * box_h * 4;
  if (tid == 0) {
    for (int s = 0; s < 4 * kMaxStages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int boxes_x = ncols / box_w, boxes_y = nrows / box_h;
  // each CTA walks its own sequence of boxes (so L2, not one hot line, serves them)
  long long t0 = clock64();
  float acc = 0.f;
  // nprod issuing threads (lane 0 of warps 0..nprod-1), each with its own ns stages and nbox / nprod boxes
  if ((tid & 31) == 0 && (tid >> 5) < nprod && mode != 1) {
    const int pw = tid >> 5;
    const int mybox = nbox / nprod;
    int issued = 0, done = 0;
    uint32_t ph = 0;
    auto issue = [&](int i) {
      const int b = (blockIdx.x * 131 + (i * nprod + pw) * 7) % (boxes_x * boxes_y);
      const int s = pw * ns + i % ns;
      mbar_arrive_expect_tx(&bar[s], box_bytes);
      tma_load_2d(smem + (size_t)s * box_bytes, &map, (b % boxes_x) * box_w, (b / boxes_x) * box_h, &bar[s]);
    };
    const int nbox = mybox;
    for (; issued < ns && issued < nbox; ++issued) issue(issued);
    while (done < nbox) {
      const int s = pw * ns + done % ns;
      mbar_wait(&bar[s], (ph >> (done % ns)) & 1u);
      ph ^= 1u << (done % ns);
      ++done;
      if (issued < nbox) {
        issue(issued);
        ++issued;
      }
    }
  } else if (tid >= 128 && mode != 0) {
    // 256 threads read 16 bytes each per step
    const int t = tid - 128, nt = 256;
    const long long total16 = (long long)nbox * box_bytes / 16 / (mode == 2 ? 2 : 1);
    const long long span16 = (long long)ncols * nrows / 4;
    long long off = ((long long)blockIdx.x * 7919 * 64) % span16;
    for (long long i = t; i < total16; i += nt) {
      float4 v;
      const float4* p = reinterpret_cast<const float4*>(base) + (off + i) % span16;
      asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
      acc += v.x + v.y + v.z + v.w;
    }
  }
  __syncthreads();
  if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
  if (acc == 1.2345f) sink[0] = acc;
}

int main() {
  // 8 MB matrix: 1024 rows x 2048 floats (L2-resident)
  const int nrows = 1024, ncols = 2048;
  float* d;
  cudaMalloc(&d, (size_t)nrows * ncols * 4);
  cudaMemset(d, 0, (size_t)nrows * ncols * 4);
  long long* dcyc;
  float* sink;
  cudaMalloc(&dcyc, 148 * 8);
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(k_tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)f;
  struct Shape { int w, h, swz; };
  const Shape shapes[] = {{32, 128, 1}, {32, 64, 1}, {32, 256, 1}, {256, 24, 0}, {256, 94, 0}};
  for (auto sh : shapes) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)ncols, (cuuint64_t)nrows};
    cuuint64_t strides[1] = {(cuuint64_t)ncols * 4};
    cuuint32_t box[2] = {(cuuint32_t)sh.w, (cuuint32_t)sh.h};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sh.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed for box %dx%d\n", sh.w, sh.h);
      continue;
    }
    const int box_bytes = sh.w * sh.h * 4;
    for (int nprod : {1, 2, 4})
    for (int ns : {1, 2, 4}) {
      if ((size_t)ns * nprod * box_bytes > 190 * 1024) continue;
      for (int mode : {0, 2}) {
        if (mode == 2 && (ns != 2 || nprod != 2)) continue;
        const int nbox = 2000;
        k_tma_rate<<<148, 384, (size_t)ns * nprod * box_bytes + 1024>>>(map, d, sh.w, sh.h, ncols, nrows, ns, nbox, mode, nprod, dcyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error: %s\n", cudaGetErrorString(e));
          return 1;
        }
        std::vector<long long> h(148);
        cudaMemcpy(h.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double bytes = (double)nbox * box_bytes * (mode == 2 ? 1.5 : 1.0);
        printf("box %3d floats x %3d rows (%s, %5.1f KB) %d issuing thread(s) x %d in flight, %s: %6.1f B/clk/SM (median CTA), %5.0f cycles per box\n",
               sh.w, sh.h, sh.swz ? "SW128" : "none ", box_bytes / 1024.0, nprod, ns,
               mode == 0 ? "TMA only      " : (mode == 1 ? "plain loads   " : "TMA + loads/2 "), bytes / h[74],
               (double)h[74] / nbox);
      }
    }
  }
  return 0;
}

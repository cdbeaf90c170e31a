// umma_rate.cu — issue rate of tcgen05.mma kind::tf32 by shape and operand
// form on every SM at once: one thread per CTA issues a train of MMAs
// (accumulating into one TMEM tile, operands rotating over the k-steps of two
// K-major SWIZZLE_128B stages), commits and waits; cycles per MMA by clock64.
// Timing only: operand contents are whatever shared memory / TMEM hold.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/umma_rate.cu -o tools/umma_rate
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
#include "../paper_2001_04179_b200/csrc/umma.cuh"

using namespace rebk;

// form 0: SS (A, B smem K-major); 1: TS (A in TMEM); 2: SS with B MN-major
// (no swizzle); 3: TS with B MN-major
template <int M, int N, int FORM>
__global__ void __launch_bounds__(128, 1) k_rate(int nmma, long long* cycles) {
  constexpr int form = FORM;
  extern __shared__ __align__(1024) float dsm[];
  float* base = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 2 * (128 + 256) * 32; i += 128) base[i] = 1.0f / (float)(1 + (i & 1023));
  if (warp == 0) umma::tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tbase;
  constexpr bool ts = form & 1, bmn = form & 2;
  constexpr uint32_t idesc = umma::idesc_tf32(M, N, false, bmn);
  float* sA[2] = {base, base + (128 + 256) * 32};
  float* sB[2] = {base + 128 * 32, base + (128 + 256) * 32 + 128 * 32};
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    for (int pass = 0; pass < 2; ++pass) {
      t0 = clock64();
      uint64_t bd0[2], ad0[2];
      for (int q = 0; q < 2; ++q) {
        bd0[q] = bmn ? umma::make_desc(umma::smem_addr(sB[q]), (uint32_t)(N / 4) * 128, 128)
                     : umma::make_desc_sw128(umma::smem_addr(sB[q]));
        ad0[q] = umma::make_desc_sw128(umma::smem_addr(sA[q]));
      }
      constexpr uint32_t bstep = bmn ? (N / 4) * 128 / 16 : 2;  // descriptor address units of 16 bytes
      for (int i = 0; i < nmma; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int s = u & 3, q = u >> 2;
          const uint64_t bd = bd0[q] + (uint64_t)(s * bstep);
          if (ts) umma::mma_tf32_ts(tmem, tmem + 256 + 8 * s + 32 * q, bd, idesc, (i | u) > 0);
          else umma::mma_tf32(tmem, ad0[q] + (uint64_t)(2 * s), bd, idesc, (i | u) > 0);
        }
      }
      umma::commit(&mbar);
      mbar_wait(&mbar, pass & 1);
      t1 = clock64();
    }
    cycles[blockIdx.x] = t1 - t0;
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<512>(tmem);
}

int main(int argc, char** argv) {
  const int allow_mn = argc > 1 ? atoi(argv[1]) : 0;
  long long* dcyc;
  cudaMalloc(&dcyc, 148 * 8);
  const size_t smem = 2 * (128 + 256) * 32 * 4 + 1024;
  const int nmma = 2048;
  auto launch = [&](int M, int N, int form, int grid) {
#define CASE(MM, NN, FF)                                                                              \
  if (M == MM && N == NN && form == FF) {                                                             \
    cudaFuncSetAttribute(k_rate<MM, NN, FF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_rate<MM, NN, FF><<<grid, 128, smem>>>(nmma, dcyc);                                              \
  }
#define CASES(FF) CASE(64, 64, FF) CASE(64, 128, FF) CASE(64, 256, FF) CASE(128, 64, FF) CASE(128, 128, FF) CASE(128, 256, FF)
    CASES(0) CASES(1) CASES(2) CASES(3)
  };
  struct Cfg { int M, N, form; };
  std::vector<Cfg> cfgs;
  for (int form = 0; form < (allow_mn ? 4 : 2); ++form)
    for (int M : {64, 128})
      for (int N : {64, 128, 256}) cfgs.push_back({M, N, form});
  for (int grid : {1, 148})
    for (auto c : cfgs) {
      launch(c.M, c.N, c.form, grid);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("M=%d N=%d form=%d: %s\n", c.M, c.N, c.form, cudaGetErrorString(e));
        return 1;
      }
      std::vector<long long> h(grid);
      cudaMemcpy(h.data(), dcyc, grid * 8, cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.end());
      const char* names[4] = {"SS Kmaj", "TS Kmaj", "SS B-MN", "TS B-MN"};
      printf("grid %3d  %s  M=%3d N=%3d : %7.1f cycles/MMA (median CTA; max %.1f)  floor M*N/256 = %d\n", grid,
             names[c.form], c.M, c.N, (double)h[grid / 2] / nmma, (double)h[grid - 1] / nmma,
             std::max(c.M, 128) * c.N / 256);
    }
  return 0;
}

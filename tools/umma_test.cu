// umma_test.cu — validates the tcgen05 kind::tf32 helpers (umma.cuh): one CTA
// computes C[128 x 64] = A[128 x K] B[K x 64] with 1x and 3x TF32 and compares
// with a double-precision host product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma_test.cu -o umma_test
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
#include "../paper_2001_04179_b200/csrc/umma.cuh"

using namespace rebk;
constexpr int M = 128, N = 64, BK = 32;

// mode 0: A K-major, B K-major (transposed on store); mode 1: A K-major, B MN-major;
// mode 2: A given as At[K][M] (m contiguous) stored MN-major, B MN-major
__global__ void __launch_bounds__(128, 1) gemm_test(const float* A, const float* B, float* C, int K, int three,
                                                    int mode, int swap) {
  extern __shared__ __align__(1024) float dsm[];
  float *sA_hi = dsm, *sA_lo = dsm + M * BK, *sB_hi = dsm + 2 * M * BK, *sB_lo = dsm + 2 * M * BK + N * BK;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) umma::tmem_alloc<64>(&tbase);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tbase;
  const uint32_t idesc = umma::idesc_tf32(M, N, mode == 2, mode == 1 || mode == 2);
  uint32_t phase = 0;
  for (int kb = 0; kb < K / BK; ++kb) {
    // A block: rows 0..127, k 0..31 (A row-major, k contiguous)
    for (int e = tid; e < M * BK; e += 128) {
      const int row = e / BK, k = e % BK;
      float hi, lo;
      umma::split_tf32(A[(size_t)row * K + kb * BK + k], hi, lo);
      if (mode == 3) hi = A[(size_t)row * K + kb * BK + k];
      const uint32_t off = (mode == 4 ? umma::kmajor_sw128_offset(row, k) : umma::kmajor_offset(row, k, M)) / 4;
      sA_hi[off] = hi;
      sA_lo[off] = lo;
    }
    // B block: k 0..BK-1, n 0..63 (B row-major, n contiguous)
    for (int e = tid; e < N * BK; e += 128) {
      const int k = e / N, n = e % N;
      float hi, lo;
      umma::split_tf32(B[(size_t)(kb * BK + k) * N + n], hi, lo);
      if (mode == 3) hi = B[(size_t)(kb * BK + k) * N + n];
      const uint32_t off = (mode == 4 ? umma::kmajor_sw128_offset(n, k)
                            : (mode == 0 || mode == 3 ? umma::kmajor_offset(n, k, N) : umma::mnmajor_offset(n, k, N))) / 4;
      sB_hi[off] = hi;
      sB_lo[off] = lo;
    }
    if (mode == 2) {  // overwrite the A tile MN-major from At = Aᵀ (row k holds all m)
      for (int e = tid; e < M * BK; e += 128) {
        const int k = e / M, m = e % M;
        float hi, lo;
        umma::split_tf32(A[(size_t)(kb * BK + k) * M + m], hi, lo);
        const uint32_t off = umma::mnmajor_offset(m, k, M) / 4;
        sA_hi[off] = hi;
        sA_lo[off] = lo;
      }
    }
    fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
    __syncthreads();
    if (tid == 0) {
      umma::fence_after_sync();
      // K-major: step = 2 chunks of LBO (M/8*128); MN-major: step = one LBO (mn/4*128)
      const bool amn = mode == 2, bmn = mode == 1 || mode == 2;
      const uint32_t lboA = amn ? (M / 4) * 128 : (M / 8) * 128, lboB = bmn ? (N / 4) * 128 : (N / 8) * 128;
      const uint32_t stA = amn ? lboA : 2 * lboA, stB = bmn ? lboB : 2 * lboB;
      for (int s = 0; s < BK / 8; ++s) {
        const bool swa = amn && swap, swb = bmn && swap;
        uint64_t ah = umma::make_desc(umma::smem_addr(sA_hi) + s * stA, swa ? 128 : lboA, swa ? lboA : 128);
        uint64_t al = umma::make_desc(umma::smem_addr(sA_lo) + s * stA, swa ? 128 : lboA, swa ? lboA : 128);
        uint64_t bh = umma::make_desc(umma::smem_addr(sB_hi) + s * stB, swb ? 128 : lboB, swb ? lboB : 128);
        uint64_t bl = umma::make_desc(umma::smem_addr(sB_lo) + s * stB, swb ? 128 : lboB, swb ? lboB : 128);
        if (mode == 4) {
          ah = umma::make_desc_sw128(umma::smem_addr(sA_hi) + 32 * s);
          al = umma::make_desc_sw128(umma::smem_addr(sA_lo) + 32 * s);
          bh = umma::make_desc_sw128(umma::smem_addr(sB_hi) + 32 * s);
          bl = umma::make_desc_sw128(umma::smem_addr(sB_lo) + 32 * s);
        }
        const bool acc = kb > 0 || s > 0;
        umma::mma_tf32(tmem, ah, bh, idesc, acc);
        if (three) {
          umma::mma_tf32(tmem, ah, bl, idesc, true);
          umma::mma_tf32(tmem, al, bh, idesc, true);
        }
      }
      umma::commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, phase);  // smem free again (and, at the end, D complete)
    phase ^= 1u;
  }
  umma::fence_after_sync();
  // epilogue: warp w reads TMEM lanes [32w, 32w+32) = rows, 64 columns
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    umma::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
    const int row = 32 * warp + (tid & 31);
    for (int i = 0; i < 16; ++i) C[(size_t)row * N + c0 + i] = v[i];
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<64>(tmem);
}

int main() {
  const int K = 256;
  std::vector<float> A((size_t)M * K), B((size_t)K * N), C((size_t)M * N);
  srand(1);
  for (auto& a : A) a = (float)rand() / RAND_MAX * 2.f - 1.f;
  for (auto& b : B) b = (float)rand() / RAND_MAX * 2.f - 1.f;
  std::vector<float> At((size_t)K * M);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < K; ++k) At[(size_t)k * M + i] = A[(size_t)i * K + k];
  float *dA, *dAt, *dB, *dC;
  cudaMalloc(&dAt, At.size() * 4);
  cudaMemcpy(dAt, At.data(), At.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(gemm_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int t = 0; t < 4; ++t) {
    const int three = t & 1, mode = t < 2 ? 0 : 4, swap = 0;
    cudaMemset(dC, 0, C.size() * 4);
    gemm_test<<<1, 128, (2 * M * BK + 2 * N * BK) * 4>>>(mode == 2 ? dAt : dA, dB, dC, K, three, mode, swap);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error: %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0, maxabs = 0, ref_norm = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[(size_t)i * K + k] * B[(size_t)k * N + j];
        maxabs = fmax(maxabs, fabs(r - C[(size_t)i * N + j]));
        ref_norm = fmax(ref_norm, fabs(r));
      }
    maxrel = maxabs / ref_norm;
    printf("swap %d mode %d %s: max |C - ref| = %.3e (relative to max |ref| %.3e: %.3e)  C[0]=%f C[last]=%f\n",
           swap, mode, three ? "3xTF32" : "1xTF32", maxabs, ref_norm, maxrel, C[0], C[C.size() - 1]);
  }
  return 0;
}

// umma_ts_test.cu — validates tcgen05 kind::tf32 with the A operand in TMEM
// ("TS" form: A [tmem], B smem descriptor): one CTA computes C[128 x 64] =
// A[128 x K] B[K x 64] with 1x and 3x TF32.  Thread t owns row t of A: it
// writes the row's 32 K values of a stage (hi, and for 3xTF32 the lo part)
// into TMEM columns with tcgen05.st (lane = row, column = k); B is staged in
// shared memory in the K-major SWIZZLE_128B layout the C5 kernel uses.
// Also times a loop of stages for the 3xTF32 SS form (A hi/lo in smem) and
// the TS form (A hi/lo in TMEM) on 148 CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma_ts_test.cu -o umma_ts_test
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
#include "../paper_2001_04179_b200/csrc/umma.cuh"

using namespace rebk;
constexpr int M = 128, N = 64, BK = 32;

__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"((uint32_t)accumulate)
      : "memory");
}

// 32 lanes x 32 columns: thread t of the warp writes lane (taddr.lane + t)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
      "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
      "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
      "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
      "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ts = 0: A hi/lo in smem (SS, as in rebk_mrhs_tc.cu); ts = 1: A hi/lo in TMEM.
// reps > 1: timing loop over the same K (result not checked)
__global__ void __launch_bounds__(128, 1) gemm_ts(const float* A, const float* B, float* C, int K, int three, int ts,
                                                  int reps, long long* cycles) {
  extern __shared__ __align__(1024) float dsm[];
  float* base = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~(uintptr_t)1023);
  float *sA_hi = base, *sA_lo = base + M * BK, *sB_hi = base + 2 * M * BK, *sB_lo = base + 2 * M * BK + N * BK;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) umma::tmem_alloc<256>(&tbase);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tbase;        // D: columns [0, 64)
  const uint32_t ta_hi = tmem + 128;  // A hi: columns [128, 160)
  const uint32_t ta_lo = tmem + 160;  // A lo: columns [160, 192)
  const uint32_t idesc = umma::idesc_tf32(M, N);
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
    for (int kb = 0; kb < K / BK; ++kb) {
      // B block -> smem (K-major SW128), split on the fly
      for (int e = tid; e < N * BK; e += 128) {
        const int k = e / N, n = e % N;
        float hi, lo;
        umma::split_tf32(B[(size_t)(kb * BK + k) * N + n], hi, lo);
        const uint32_t off = umma::kmajor_sw128_offset(n, k) / 4;
        sB_hi[off] = B[(size_t)(kb * BK + k) * N + n];
        sB_lo[off] = lo;
      }
      // A block: thread tid = row
      float hi[BK], lo[BK];
#pragma unroll
      for (int k = 0; k < BK; ++k) {
        float h;
        const float a = A[(size_t)tid * K + kb * BK + k];
        umma::split_tf32(a, h, lo[k]);
        hi[k] = a;  // raw value as "hi": the MMA truncates to tf32
      }
      if (ts) {
        const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
        tmem_st32(ta_hi + lane_base, hi);
        tmem_st32(ta_lo + lane_base, lo);
        tmem_wait_st();
      } else {
#pragma unroll
        for (int k = 0; k < BK; ++k) {
          const uint32_t off = umma::kmajor_sw128_offset(tid, k) / 4;
          sA_hi[off] = hi[k];
          sA_lo[off] = lo[k];
        }
      }
      fence_proxy_async();
      umma::fence_before_sync();
      __syncthreads();
      if (tid == 0) {
        umma::fence_after_sync();
        for (int s = 0; s < BK / 8; ++s) {
          const uint64_t bh = umma::make_desc_sw128(umma::smem_addr(sB_hi) + 32 * s);
          const uint64_t bl = umma::make_desc_sw128(umma::smem_addr(sB_lo) + 32 * s);
          const bool acc = rep > 0 || kb > 0 || s > 0;
          if (ts) {
            mma_tf32_ts(tmem, ta_hi + 8 * s, bh, idesc, acc);
            if (three) {
              mma_tf32_ts(tmem, ta_hi + 8 * s, bl, idesc, true);
              mma_tf32_ts(tmem, ta_lo + 8 * s, bh, idesc, true);
            }
          } else {
            const uint64_t ah = umma::make_desc_sw128(umma::smem_addr(sA_hi) + 32 * s);
            const uint64_t al = umma::make_desc_sw128(umma::smem_addr(sA_lo) + 32 * s);
            umma::mma_tf32(tmem, ah, bh, idesc, acc);
            if (three) {
              umma::mma_tf32(tmem, ah, bl, idesc, true);
              umma::mma_tf32(tmem, al, bh, idesc, true);
            }
          }
        }
        umma::commit(&mbar);
      }
      __syncwarp();
      mbar_wait(&mbar, phase);
      phase ^= 1u;
    }
  if (tid == 0 && cycles) cycles[blockIdx.x] = clock64() - t0;
  umma::fence_after_sync();
  if (blockIdx.x == 0) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      umma::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      const int row = 32 * warp + (tid & 31);
      for (int i = 0; i < 16; ++i) C[(size_t)row * N + c0 + i] = v[i];
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<256>(tmem);
}

int main() {
  const int K = 256;
  std::vector<float> A((size_t)M * K), B((size_t)K * N), C((size_t)M * N);
  srand(1);
  for (auto& a : A) a = (float)rand() / RAND_MAX * 2.f - 1.f;
  for (auto& b : B) b = (float)rand() / RAND_MAX * 2.f - 1.f;
  float *dA, *dB, *dC;
  long long* dcyc;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMalloc(&dcyc, 148 * 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = (2 * M * BK + 2 * N * BK) * 4 + 1024;
  cudaFuncSetAttribute(gemm_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int rc = 0;
  for (int t = 0; t < 4; ++t) {
    const int three = t & 1, ts = t >> 1;
    cudaMemset(dC, 0, C.size() * 4);
    gemm_ts<<<1, 128, smem>>>(dA, dB, dC, K, three, ts, 1, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error (ts=%d three=%d): %s\n", ts, three, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double maxabs = 0, ref_norm = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[(size_t)i * K + k] * B[(size_t)k * N + j];
        maxabs = fmax(maxabs, fabs(r - C[(size_t)i * N + j]));
        ref_norm = fmax(ref_norm, fabs(r));
      }
    const double rel = maxabs / ref_norm;
    const bool ok = rel < (three ? 1e-5 : 3e-3);
    rc |= !ok;
    printf("%s A in %s: max |C - ref| / max|ref| = %.3e  %s\n", three ? "3xTF32" : "1xTF32", ts ? "TMEM" : "smem",
           rel, ok ? "ok" : "FAIL");
  }
  return rc;
}

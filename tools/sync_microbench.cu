// sync_microbench.cu — measures the grid-wide exchange primitives the REBK
// kernel design depends on (not part of the product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_mb tools/sync_microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void bar_arrive_wait(unsigned long long* bar, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
    unsigned long long v;
    do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory"); } while (v < target);
  }
  __syncthreads();
}

// 1. counter barrier only
__global__ void k_barrier(unsigned long long* bar, int iters) {
  unsigned long long t = 0;
  for (int i = 0; i < iters; ++i) { t += gridDim.x; bar_arrive_wait(bar, t); }
}

// 2. flag all-gather: every CTA publishes seq, then polls all G flags (one thread per flag)
__global__ void k_flags(unsigned* flags, int iters) {
  const int G = gridDim.x;
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"(i) : "memory");
    for (int q = threadIdx.x; q < G; q += blockDim.x) {
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q * 32) : "memory"); } while ((int)(v - i) < 0);
    }
    __syncthreads();
  }
}

// 3. partial write + barrier + reduce-scatter + barrier + all-gather (the v1 exchange)
__global__ void k_rs_ag(unsigned long long* bar, double* part, double* out, int n, int iters) {
  const int G = gridDim.x, g = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  unsigned long long t = 0;
  __shared__ double sv[1024];
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    for (int e = threadIdx.x; e < n; e += blockDim.x) __stcg(part + (size_t)e * G + g, (double)(e + g + i));
    t += G; bar_arrive_wait(bar, t);
    for (int e = g * W + warp; e < n; e += G * W) {
      double s = 0;
      for (int q = lane; q < G; q += 32) s += __ldcg(part + (size_t)e * G + q);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
      if (lane == 0) __stcg(out + e, s);
    }
    t += G; bar_arrive_wait(bar, t);
    for (int e = threadIdx.x; e < n; e += blockDim.x) sv[e] = __ldcg(out + e);
    __syncthreads();
    acc += sv[(i * 7) % n];
  }
  if (acc == 12345.678) out[0] = acc;
}

// 4. fixed-point red.add (L limbs per value, padded to spread L2 slices) + barrier + read
__global__ void k_red(unsigned long long* bar, unsigned long long* acc, int n, int limbs, int pad, int iters) {
  const int G = gridDim.x;
  unsigned long long t = 0;
  __shared__ double sv[1024];
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned long long* buf = acc + (size_t)(i & 1) * n * limbs * pad;
    for (int e = threadIdx.x; e < n * limbs; e += blockDim.x)
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(buf + (size_t)e * pad), "l"((unsigned long long)(e + blockIdx.x)) : "memory");
    t += G; bar_arrive_wait(bar, t);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      unsigned long long v = 0;
      for (int l = 0; l < limbs; ++l) v += __ldcg(buf + (size_t)(e * limbs + l) * pad);
      sv[e] = (double)v;
    }
    // zero the other parity buffer (own slice) for the next-next use
    unsigned long long* ob = acc + (size_t)((i + 1) & 1) * n * limbs * pad;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * limbs; e += G * blockDim.x) __stcg(ob + (size_t)e * pad, 0ull);
    __syncthreads();
    s += sv[i % n];
  }
  if (s == 1.5) acc[0] = 1;
}

// 5. empty persistent loop with __syncthreads only (floor)
__global__ void k_local(int iters, int* out) {
  int v = 0;
  for (int i = 0; i < iters; ++i) { __syncthreads(); v += threadIdx.x; }
  if (v == -1) *out = v;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  int G = 148, T = 256, iters = 20000;
  unsigned long long* bar; CK(cudaMalloc(&bar, 8));
  unsigned* flags; CK(cudaMalloc(&flags, 4 * 32 * 256)); CK(cudaMemset(flags, 0, 4 * 32 * 256));
  double *part, *out; CK(cudaMalloc(&part, 8 * 1024 * 256)); CK(cudaMalloc(&out, 8 * 1024));
  unsigned long long* acc; CK(cudaMalloc(&acc, 8ull * 2 * 1200 * 32)); CK(cudaMemset(acc, 0, 8ull * 2 * 1200 * 32));
  int* dummy; CK(cudaMalloc(&dummy, 4));
  for (int g : {16, 64, 148}) {
    void* args1[] = {&bar, &iters};
    float ms = timeit([&] { cudaMemset(bar, 0, 8); cudaLaunchCooperativeKernel((void*)k_barrier, g, T, args1); });
    printf("grid=%3d counter barrier: %.3f us\n", g, ms * 1e3 / iters);
    void* args2[] = {&flags, &iters};
    cudaMemset(flags, 0, 4 * 32 * 256);
    ms = timeit([&] { cudaMemset(flags, 0, 4 * 32 * 256); cudaLaunchCooperativeKernel((void*)k_flags, g, T, args2); });
    printf("grid=%3d flag all-gather: %.3f us\n", g, ms * 1e3 / iters);
    int n = 400;
    void* args3[] = {&bar, &part, &out, &n, &iters};
    ms = timeit([&] { cudaMemset(bar, 0, 8); cudaLaunchCooperativeKernel((void*)k_rs_ag, g, T, args3); });
    printf("grid=%3d RS+AG (n=400) 2 barriers: %.3f us\n", g, ms * 1e3 / iters);
    for (int limbs : {1, 2, 3}) for (int pad : {1, 16, 32}) {
      void* args4[] = {&bar, &acc, &n, &limbs, &pad, &iters};
      ms = timeit([&] { cudaMemset(bar, 0, 8); cudaLaunchCooperativeKernel((void*)k_red, g, T, args4); });
      printf("grid=%3d red fixed-point n=400 limbs=%d pad=%2d + barrier: %.3f us\n", g, limbs, pad, ms * 1e3 / iters);
    }
  }
  void* args5[] = {&iters, &dummy};
  float ms = timeit([&] { cudaLaunchKernel((void*)k_local, 148, T, args5, 0, 0); });
  printf("local syncthreads loop: %.3f us\n", ms * 1e3 / iters);
  return 0;
}

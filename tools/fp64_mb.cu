// fp64_mb.cu — DFMA latency/throughput and LDS.128 throughput on one SM (not product code)
#include <cstdio>
__global__ void lat(double* o, int n) {
  double a = o[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  if (threadIdx.x == 0) { o[100] = (double)(t1 - t0) / n; }
  o[threadIdx.x + 200] = a;
}
template <int CH>
__global__ void thr(double* o, int n) {
  double a[CH];
  for (int j = 0; j < CH; ++j) a[j] = o[threadIdx.x % 32 + j];
  double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < CH; ++j) a[j] = fma(a[j], b, c);
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int j = 0; j < CH; ++j) s += a[j];
  if (threadIdx.x == 0) o[100] = (double)(t1 - t0) / n / CH;  // cycles per DFMA per thread
  o[threadIdx.x + 300] = s;
}
__global__ void lds(double* o, int n) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double2 acc = make_double2(0, 0);
  const double2* p = reinterpret_cast<const double2*>(sm);
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double2 v = p[(threadIdx.x + i * 37) & 2047];
    acc.x += v.x; acc.y += v.y;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) o[100] = (double)(t1 - t0) / n;
  o[threadIdx.x + 300] = acc.x + acc.y;
}
int main() {
  double* d; cudaMalloc(&d, 8 * 4096); cudaMemset(d, 0, 8 * 4096);
  double h;
  lat<<<1, 32>>>(d, 10000); cudaMemcpy(&h, d + 100, 8, cudaMemcpyDeviceToHost); printf("DFMA dependent latency: %.2f cycles\n", h);
  for (int T : {32, 128, 256, 512, 1024}) {
    thr<8><<<1, T>>>(d, 2000); cudaMemcpy(&h, d + 100, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 chains, %4d threads/SM: %.3f cycles per DFMA per thread => %.1f DFMA/clk/SM\n", T, h, T / h);
  }
  for (int T : {128, 256, 512, 1024}) {
    lds<<<1, T>>>(d, 2000); cudaMemcpy(&h, d + 100, 8, cudaMemcpyDeviceToHost);
    printf("LDS.128 %4d threads: %.2f cycles/iter => %.1f B/clk\n", T, h, T * 16 / h);
  }
  return 0;
}

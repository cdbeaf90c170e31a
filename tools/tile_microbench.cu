// tile_microbench.cu — time the fast path's shared-memory tile products in
// isolation (clock64 per call, one CTA per SM), to separate compute cost from
// synchronisation cost.  Not part of the product.
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;

__global__ void __launch_bounds__(kThreads, 1) k_tiles(int R, int C, int ld, int which, int reps, long long* out, double* sink) {
  extern __shared__ __align__(128) double sm[];
  double* T = sm;
  double* v = T + (size_t)R * ld + 16;
  double* red = v + ((R > C ? R : C) + 16);
  double* o = red + 2 * kThreads;
  for (int i = threadIdx.x; i < R * ld; i += kThreads) T[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < (R > C ? R : C) + 2; i += kThreads) v[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (which == 0) colsum2(T, ld, R, C, v, red, [&](int c, double a) { o[c] = a; });
    else rowdot2(T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = (t1 - t0) / reps; sink[blockIdx.x] = o[0]; }
}

int main() {
  long long* d; double* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 8 * 1024);
  cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct { int R, C, ld; const char* what; } cfgs[] = {
    {34, 200, 200, "C2 col tile (G=120)"}, {200, 84, 86, "C2 row tile (G=120)"},
    {28, 200, 200, "C2 col tile (G=148)"}, {200, 68, 70, "C2 row tile (G=148)"},
    {125, 100, 100, "C1 col tile (G=16)"}, {100, 32, 34, "C1 row tile (G=16)"}};
  for (auto& c : cfgs) for (int which = 0; which < 2; ++which) {
    size_t smem = ((size_t)c.R * c.ld + 16 + (c.R > c.C ? c.R : c.C) + 16 + 2 * 256 + 512) * 8;
    k_tiles<<<148, kThreads, smem>>>(c.R, c.C, c.ld, which, 50, d, s);
    long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    double bytes = (double)c.R * c.C * 8;
    printf("%-22s %-8s R=%3d C=%3d: %6lld cycles  (%.1f B/clk smem) %s\n", c.what, which ? "rowdot2" : "colsum2", c.R, c.C, h[0], bytes / h[0], e ? cudaGetErrorString(e) : "");
  }
  return 0;
}

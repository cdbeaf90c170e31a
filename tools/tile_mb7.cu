// tile_mb7.cu — what caps the tile products at ~60 B/clk?  streaming reads of
// a 200 KB smem tile with: DADD only / DFMA / DFMA + broadcast LDS.64 /
// 2 rows per thread in flight.
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;
template <int NT>
__global__ void __launch_bounds__(NT, 1) k(int n2, int which, int reps, long long* out, double* sink) {
  extern __shared__ __align__(128) double sm[];
  double2* T = reinterpret_cast<double2*>(sm);
  double* v = sm + 2 * n2 + 64;
  for (int i = threadIdx.x; i < 2 * n2; i += NT) sm[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 512; i += NT) v[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  double2 a = make_double2(0, 0), b = a;
  const double c = v[threadIdx.x & 7];
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (which == 0) {
      for (int i = threadIdx.x; i < n2; i += NT) { double2 t = T[i]; a.x += t.x; a.y += t.y; }
    } else if (which == 1) {
      for (int i = threadIdx.x; i < n2; i += NT) { double2 t = T[i]; a.x = fma(t.x, c, a.x); a.y = fma(t.y, c, a.y); }
    } else if (which == 2) {
      for (int i = threadIdx.x; i < n2; i += NT) { double2 t = T[i]; const double w = v[i / 100]; a.x = fma(t.x, w, a.x); a.y = fma(t.y, w, a.y); }
    } else if (which == 3) {
      int i = threadIdx.x;
      for (; i + NT < n2; i += 2 * NT) { double2 t = T[i], u = T[i + NT]; a.x = fma(t.x, c, a.x); a.y = fma(t.y, c, a.y); b.x = fma(u.x, c, b.x); b.y = fma(u.y, c, b.y); }
      if (i < n2) { double2 t = T[i]; a.x = fma(t.x, c, a.x); a.y = fma(t.y, c, a.y); }
    } else {
      int i = threadIdx.x;
#pragma unroll 4
      for (; i < n2; i += NT) { double2 t = T[i]; a.x = fma(t.x, c, a.x); a.y = fma(t.y, c, a.y); }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
  sink[blockIdx.x * NT + threadIdx.x] = a.x + a.y + b.x + b.y;
}
template <int NT> void run() {
  long long* d; double* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 8 * 148 * 1024);
  cudaFuncSetAttribute(k<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  const int n2 = 12000;  // 192 KB
  const char* nm[] = {"DADD", "DFMA", "DFMA+bcastLDS", "DFMA 2-in-flight", "DFMA unroll4"};
  for (int w = 0; w < 5; ++w) {
    k<NT><<<148, NT, (2 * n2 + 64 + 512) * 8>>>(n2, w, 50, d, s);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("NT=%d %-18s %6lld cycles (%.1f B/clk) %s\n", NT, nm[w], h, 192000.0 / h, cudaGetErrorString(cudaGetLastError()));
  }
}
int main() { run<256>(); run<512>(); run<1024>(); return 0; }

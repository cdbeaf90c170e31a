// tile_mb3.cu — where does the fixed per-call cost of the tile products come from?
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;
__global__ void __launch_bounds__(kThreads, 1) k(int R, int C, int ld, int which, int reps, long long* out, double* sink) {
  extern __shared__ __align__(128) double sm[];
  double* T = sm; double* v = T + (size_t)R * ld + 16; double* red = v + 512; double* o = red + 2 * kThreads;
  for (int i = threadIdx.x; i < R * ld; i += kThreads) T[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 512; i += kThreads) v[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (which == 0) { }
    else if (which == 1) colsum2(T, ld, R, C, v, red, [&](int c, double a) { o[c] = a; });
    else if (which == 2) rowdot2(T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    else if (which == 3) { // raw streaming read of the tile, 256 threads, LDS.128
      const double2* p = reinterpret_cast<const double2*>(T); double2 a = make_double2(0,0);
      for (int i = threadIdx.x; i < R * ld / 2; i += kThreads) { double2 t = p[i]; a.x += t.x; a.y += t.y; }
      o[threadIdx.x] = a.x + a.y;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = (t1 - t0) / reps; sink[blockIdx.x] = o[0]; }
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 8 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* nm[] = {"empty", "colsum2", "rowdot2", "stream"};
  int Rs[] = {1, 8, 28, 200}, Cs[] = {200, 200, 200, 68};
  for (int i = 0; i < 4; ++i) for (int w = 0; w < 4; ++w) {
    int R = Rs[i], C = Cs[i], ld = C + 2;
    size_t smem = ((size_t)R * ld + 16 + 512 + 2 * 256 + 512) * 8;
    for (int grid : {1, 148}) {
      k<<<grid, kThreads, smem>>>(R, C, ld, w, 200, d, s);
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("grid %3d R=%3d C=%3d %-8s %6lld cycles\n", grid, R, C, nm[w], h);
    }
  }
  return 0;
}

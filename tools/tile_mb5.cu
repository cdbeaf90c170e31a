// tile_mb5.cu — split-kernel tile products at 256 vs 512 threads (colsum2/rowdot2<NT>)
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;
template <int NT>
__global__ void __launch_bounds__(NT, 1) k(int R, int C, int ld, int which, int reps, long long* out, double* sink) {
  extern __shared__ __align__(128) double sm[];
  double* T = sm; double* v = T + (size_t)R * ld + 16; double* red = v + 512; double* o = red + 2 * NT;
  for (int i = threadIdx.x; i < R * ld; i += NT) T[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 512; i += NT) v[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (which == 0) colsum2<NT>(T, ld, R, C, v, red, [&](int c, double a) { o[c] = a; });
    else if (which == 1) rowdot2<NT>(T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    else {
      const double2* p = reinterpret_cast<const double2*>(T); double2 a = make_double2(0, 0);
      for (int i = threadIdx.x; i < R * ld / 2; i += NT) { double2 t = p[i]; a.x += t.x; a.y += t.y; }
      o[threadIdx.x] = a.x + a.y;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = (t1 - t0) / reps; sink[blockIdx.x] = o[0]; }
}
template <int NT> void run(int R, int C, int ld, const char* nm) {
  long long* d; double* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 8 * 1024);
  cudaFuncSetAttribute(k<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int w = 0; w < 3; ++w) {
    size_t smem = ((size_t)R * ld + 16 + 512 + 2 * NT + 1024) * 8;
    k<NT><<<148, NT, smem>>>(R, C, ld, w, 100, d, s);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("NT=%d %-18s R=%3d C=%3d %-7s %6lld cycles (%.1f B/clk) %s\n", NT, nm, R, C, w == 0 ? "colsum" : w == 1 ? "rowdot" : "stream", h, (double)R * C * 8 / h, cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  run<256>(125, 200, 200, "split col tile"); run<512>(125, 200, 200, "split col tile");
  run<256>(200, 114, 114, "split row tile"); run<512>(200, 114, 114, "split row tile");
  return 0;
}

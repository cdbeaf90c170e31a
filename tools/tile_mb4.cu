// tile_mb4.cu — tile products with per-run precomputed thread mappings
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;

struct ColMap { int CP, RG, cp, rg; };
struct RowMap { int L, sub, rsub, rpp, CPf; };
__device__ ColMap make_colmap(int R, int C) {
  ColMap m; m.CP = (C + 1) >> 1; m.RG = kThreads / m.CP; if (m.RG > R) m.RG = R > 0 ? R : 1;
  m.cp = threadIdx.x % m.CP; m.rg = threadIdx.x / m.CP; return m;
}
__device__ RowMap make_rowmap(int R, int C) {
  RowMap m; m.CPf = C >> 1; int L = pow2floor(kThreads / R); const int lmax = m.CPf >= 1 ? pow2floor(m.CPf) : 1;
  L = L > 32 ? 32 : L; L = L > lmax ? lmax : L; m.L = L; m.sub = threadIdx.x % L; m.rsub = threadIdx.x / L; m.rpp = kThreads / L; return m;
}
// colsum with map; no block reduction when RG == 1
template <typename Epi>
__device__ __forceinline__ void colsum_m(const ColMap& mp, const double* __restrict__ T, int ld, int R, int C,
                                         const double* __restrict__ v, double* red, Epi epi) {
  double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
  if (mp.rg < mp.RG) {
    const double* col = T + 2 * mp.cp;
    const int RG = mp.RG;
    int r = mp.rg;
    for (; r + 3 * RG < R; r += 4 * RG) {
      const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * ld);
      const double2 t1 = *reinterpret_cast<const double2*>(col + (size_t)(r + RG) * ld);
      const double2 t2 = *reinterpret_cast<const double2*>(col + (size_t)(r + 2 * RG) * ld);
      const double2 t3 = *reinterpret_cast<const double2*>(col + (size_t)(r + 3 * RG) * ld);
      const double v0 = v[r], v1 = v[r + RG], v2 = v[r + 2 * RG], v3 = v[r + 3 * RG];
      a0.x = fma(t0.x, v0, a0.x); a0.y = fma(t0.y, v0, a0.y);
      a1.x = fma(t1.x, v1, a1.x); a1.y = fma(t1.y, v1, a1.y);
      a2.x = fma(t2.x, v2, a2.x); a2.y = fma(t2.y, v2, a2.y);
      a3.x = fma(t3.x, v3, a3.x); a3.y = fma(t3.y, v3, a3.y);
    }
    for (; r < R; r += RG) {
      const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * ld);
      const double v0 = v[r];
      a0.x = fma(t0.x, v0, a0.x); a0.y = fma(t0.y, v0, a0.y);
    }
  }
  const double sx = (a0.x + a1.x) + (a2.x + a3.x), sy = (a0.y + a1.y) + (a2.y + a3.y);
  if (mp.RG == 1) {
    if (mp.rg < 1) { epi(2 * mp.cp, sx); if (2 * mp.cp + 1 < C) epi(2 * mp.cp + 1, sy); }
    return;
  }
  if (mp.rg < mp.RG) { red[mp.rg * 2 * mp.CP + 2 * mp.cp] = sx; red[mp.rg * 2 * mp.CP + 2 * mp.cp + 1] = sy; }
  __syncthreads();
  if (threadIdx.x < C) {
    double s = 0.0;
    for (int q = 0; q < mp.RG; ++q) s += red[q * 2 * mp.CP + threadIdx.x];
    epi(threadIdx.x, s);
  }
}
template <typename Epi>
__device__ __forceinline__ void rowdot_m(const RowMap& mp, const double* __restrict__ T, int ld, int R, int C,
                                         const double* __restrict__ v, Epi epi) {
  const double2* v2 = reinterpret_cast<const double2*>(v);
  const int L = mp.L;
  for (int r0 = 0; r0 < R; r0 += mp.rpp) {
    const int r = r0 + mp.rsub;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    if (r < R) {
      const double2* row = reinterpret_cast<const double2*>(T + (size_t)r * ld);
      int q = mp.sub;
      for (; q + L < mp.CPf; q += 2 * L) {
        const double2 t0 = row[q], t1 = row[q + L];
        const double2 w0 = v2[q], w1 = v2[q + L];
        c0 = fma(t0.x, w0.x, c0); c1 = fma(t0.y, w0.y, c1); c2 = fma(t1.x, w1.x, c2); c3 = fma(t1.y, w1.y, c3);
      }
      if (q < mp.CPf) { const double2 t0 = row[q], w0 = v2[q]; c0 = fma(t0.x, w0.x, c0); c1 = fma(t0.y, w0.y, c1); }
    }
    double acc = (c0 + c1) + (c2 + c3);
    for (int off = L / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (mp.sub == 0 && r < R) epi(r, acc);
  }
}

__global__ void __launch_bounds__(kThreads, 1) k(int R, int C, int ld, int which, int reps, long long* out, double* sink) {
  extern __shared__ __align__(128) double sm[];
  double* T = sm; double* v = T + (size_t)R * ld + 16; double* red = v + 512; double* o = red + 2 * kThreads;
  for (int i = threadIdx.x; i < R * ld; i += kThreads) T[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 512; i += kThreads) v[i] = 1.0 + 1e-3 * i;
  const ColMap cm = make_colmap(R, C); const RowMap rm = make_rowmap(R, C);
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (which == 0) colsum_m(cm, T, ld, R, C, v, red, [&](int c, double a) { o[c] = a; });
    else rowdot_m(rm, T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = (t1 - t0) / reps; sink[blockIdx.x] = o[0]; }
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 8 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int Rs[] = {1, 28, 200, 100, 125}, Cs[] = {200, 200, 68, 94, 100};
  for (int i = 0; i < 5; ++i) for (int w = 0; w < 2; ++w) {
    int R = Rs[i], C = Cs[i], ld = ((C + 1) & ~1); if (ld % 4 == 0) ld += 2;
    size_t smem = ((size_t)R * ld + 16 + 512 + 2 * 256 + 512) * 8;
    k<<<148, kThreads, smem>>>(R, C, ld, w, 200, d, s);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("R=%3d C=%3d %-8s %6lld cycles (%.1f B/clk)\n", R, C, w ? "rowdot" : "colsum", h, (double)R * C * 8 / h);
  }
  return 0;
}

// tile_microbench2.cu — candidate tile products with batched loads, and the
// flat LL128 exchange (no clusters).  Not product code.
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;

template <int B, typename Epi>
__device__ __forceinline__ void colsum3(const double* __restrict__ T, int ld, int R, int C,
                                        const double* __restrict__ v, double* red, Epi epi) {
  const int tid = threadIdx.x;
  const int CP = (C + 1) >> 1;
  int RG = kThreads / CP;
  if (RG > R) RG = R > 0 ? R : 1;
  const int cp = tid % CP, rg = tid / CP;
  double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
  if (rg < RG) {
    const double* col = T + 2 * cp;
    for (int r0 = rg; r0 < R; r0 += B * RG) {
      double2 t[B];
      double w[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int r = r0 + j * RG;
        if (r < R) { t[j] = *reinterpret_cast<const double2*>(col + (size_t)r * ld); w[j] = v[r]; }
        else { t[j] = make_double2(0, 0); w[j] = 0.0; }
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        acc[j & 1].x = fma(t[j].x, w[j], acc[j & 1].x);
        acc[j & 1].y = fma(t[j].y, w[j], acc[j & 1].y);
      }
    }
  }
  const double sx = acc[0].x + acc[1].x, sy = acc[0].y + acc[1].y;
  __syncthreads();
  if (rg < RG) { red[rg * 2 * CP + 2 * cp] = sx; red[rg * 2 * CP + 2 * cp + 1] = sy; }
  __syncthreads();
  for (int c = tid; c < C; c += kThreads) {
    double s = 0.0;
    for (int q = 0; q < RG; ++q) s += red[q * 2 * CP + c];
    epi(c, s);
  }
}

template <int B, typename Epi>
__device__ __forceinline__ void rowdot3(const double* __restrict__ T, int ld, int R, int C,
                                        const double* __restrict__ v, Epi epi) {
  const int tid = threadIdx.x;
  const int CPf = C >> 1;
  int L = pow2floor(kThreads / R);
  const int lmax = CPf >= 1 ? pow2floor(CPf) : 1;
  L = L > 32 ? 32 : L;
  L = L > lmax ? lmax : L;
  const int sub = tid % L, rsub = tid / L, rpp = kThreads / L;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  for (int rr = 0; rr < R; rr += rpp) {
    const int r = rr + rsub;
    double c0 = 0, c1 = 0;
    if (r < R) {
      const double2* row = reinterpret_cast<const double2*>(T + (size_t)r * ld);
      for (int q0 = sub; q0 < CPf; q0 += B * L) {
        double2 t[B], w[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int q = q0 + j * L;
          if (q < CPf) { t[j] = row[q]; w[j] = v2[q]; } else { t[j] = make_double2(0, 0); w[j] = t[j]; }
        }
#pragma unroll
        for (int j = 0; j < B; ++j) { c0 = fma(t[j].x, w[j].x, c0); c1 = fma(t[j].y, w[j].y, c1); }
      }
      if ((C & 1) && sub == (CPf % L)) c1 = fma(T[(size_t)r * ld + C - 1], v[C - 1], c1);
    }
    double acc = c0 + c1;
    for (int off = L / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (sub == 0 && r < R) epi(r, acc);
  }
}

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
    else if (which == 1) rowdot2(T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    else if (which == 2) colsum3<8>(T, ld, R, C, v, red, [&](int c, double a) { o[c] = a; });
    else if (which == 3) rowdot3<8>(T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    else if (which == 4) colsum3<16>(T, ld, R, C, v, red, [&](int c, double a) { o[c] = a; });
    else rowdot3<16>(T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = (t1 - t0) / reps; sink[blockIdx.x] = o[0]; }
}

// flat LL exchange: part[g][e] -> slice owners -> fin[e] -> everyone
__global__ void k_flat(LLWord* part, LLWord* fin, int ne, int iters, long long* out, double* sink) {
  __shared__ double s_tmp[4096];
  __shared__ double s_out[1024];
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int e0 = (int)((long long)ne * g / G), e1 = (int)((long long)ne * (g + 1) / G), nmy = e1 - e0;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    const unsigned long long seq = it;
    for (int e = tid; e < ne; e += kThreads) st_ll(part + (size_t)g * ne + e, 1.0 + e + g + acc * 1e-30, seq);
    for (int t = tid; t < G * nmy; t += kThreads) { int q = t / nmy, e = t - q * nmy; s_tmp[t] = poll_ll(part + (size_t)q * ne + e0 + e, seq); }
    __syncthreads();
    { const int lane = tid & 31, warp = tid >> 5;
      for (int e = warp; e < nmy; e += kWarps) {
        double s = 0; for (int q = lane; q < G; q += 32) s += s_tmp[q * nmy + e];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
        if (lane == 0) st_ll(fin + e0 + e, s, seq);
      } }
    for (int e = tid; e < ne; e += kThreads) s_out[e] = poll_ll(fin + e, seq);
    __syncthreads();
    acc += s_out[it % ne];
  }
  long long t1 = clock64();
  if (tid == 0) { out[g] = (t1 - t0) / iters; sink[g] = acc; }
}

int main(int argc, char** argv) {
  bool only_x = argc > 1;
  long long* d; double* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 8 * 1024);
  cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct { int R, C, ld; const char* what; } cfgs[] = {
    {28, 200, 200, "C2 col tile (G=148)"}, {200, 68, 70, "C2 row tile (G=148)"},
    {125, 100, 100, "C1 col tile (G=16)"}, {100, 32, 34, "C1 row tile (G=16)"}};
  const char* names[] = {"colsum2", "rowdot2", "colsum3<8>", "rowdot3<8>", "colsum3<16>", "rowdot3<16>"};
  if (!only_x) for (auto& c : cfgs) for (int which = 0; which < 6; ++which) {
    size_t smem = ((size_t)c.R * c.ld + 16 + (c.R > c.C ? c.R : c.C) + 16 + 2 * 256 + 512) * 8;
    k_tiles<<<148, kThreads, smem>>>(c.R, c.C, c.ld, which, 50, d, s);
    long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double bytes = (double)c.R * c.C * 8;
    printf("%-22s %-12s R=%3d C=%3d: %6lld cycles  (%.1f B/clk)\n", c.what, names[which], c.R, c.C, h[0], bytes / h[0]);
  }
  LLWord *part, *fin; cudaMalloc(&part, 16 * 148 * 1024); cudaMalloc(&fin, 16 * 1024);
  for (int ne : {200, 400}) for (int G : {64, 120, 148}) {
    cudaMemset(part, 0, 16 * 148 * 1024); cudaMemset(fin, 0, 16 * 1024);
    int iters = 5000;
    void* args[] = {&part, &fin, &ne, &iters, &d, &s};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_flat, G, kThreads, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("flat LL exchange G=%3d ne=%3d: %.3f us per exchange %s\n", G, ne, ms * 1e3 / iters, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}

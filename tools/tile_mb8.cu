// tile_mb8.cu — the split kernel's tile products in isolation (no TMA, no
// exchange): rowdot2 / rowdot2x / colsum2h on the C2 half-tile shapes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tile_mb8.cu -o tile_mb8
#include <cstdio>

#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;
constexpr int NT = 512;

// compile-time L, fully unrolled pair loop (MAXQ pairs per lane), two rows per thread
template <int L, int MAXQ, typename Epi>
__device__ __forceinline__ void rowdot_ct(const double* __restrict__ T, int ld, int R, int C, const double* __restrict__ v,
                                          Epi epi) {
  const int tid = threadIdx.x;
  const int CPf = C >> 1;
  const int sub = tid % L, rsub = tid / L;
  constexpr int rpp = NT / L;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  for (int r0 = 0; r0 < R; r0 += 2 * rpp) {
    const int ra = r0 + rsub, rb = ra + rpp;
    const bool ha = ra < R, hb = rb < R;
    const double2* rowa = reinterpret_cast<const double2*>(T + (size_t)(ha ? ra : 0) * ld);
    const double2* rowb = reinterpret_cast<const double2*>(T + (size_t)(hb ? rb : 0) * ld);
    double2 w[MAXQ], s[MAXQ], t[MAXQ];
#pragma unroll
    for (int i = 0; i < MAXQ; ++i) {
      const int q = sub + i * L;
      const bool in = q < CPf;
      w[i] = in ? v2[q] : make_double2(0.0, 0.0);
      s[i] = (in && ha) ? rowa[q] : make_double2(0.0, 0.0);
      t[i] = (in && hb) ? rowb[q] : make_double2(0.0, 0.0);
    }
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int i = 0; i < MAXQ; ++i) {
      a0 = fma(s[i].x, w[i].x, a0);
      a1 = fma(s[i].y, w[i].y, a1);
      b0 = fma(t[i].x, w[i].x, b0);
      b1 = fma(t[i].y, w[i].y, b1);
    }
    double acc = a0 + a1, bcc = b0 + b1;
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, off);
      bcc += __shfl_xor_sync(0xffffffffu, bcc, off);
    }
    if (sub == 0 && ha) epi(ra, acc);
    if (sub == 0 && hb) epi(rb, bcc);
  }
}

// colsum with 8 rows in flight per thread, chunked (consecutive) rows per thread
template <typename Epi>
__device__ __forceinline__ void colsum_u8(const double* __restrict__ T, int ld, int R, int C, const double* __restrict__ v,
                                          double* red, Epi epi) {
  const int tid = threadIdx.x;
  const int CP = (C + 1) >> 1;
  int RG = NT / CP;
  if (RG > R) RG = R;
  const int cp = tid % CP, rg = tid / CP;
  double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
  if (rg < RG) {
    const double* col = T + 2 * cp;
    int r = rg;
    for (; r + 7 * RG < R; r += 8 * RG) {
      double2 t[8];
      double w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        t[i] = *reinterpret_cast<const double2*>(col + (size_t)(r + i * RG) * ld);
        w[i] = v[r + i * RG];
      }
#pragma unroll
      for (int i = 0; i < 8; i += 4) {
        a0.x = fma(t[i].x, w[i], a0.x);
        a0.y = fma(t[i].y, w[i], a0.y);
        a1.x = fma(t[i + 1].x, w[i + 1], a1.x);
        a1.y = fma(t[i + 1].y, w[i + 1], a1.y);
        a2.x = fma(t[i + 2].x, w[i + 2], a2.x);
        a2.y = fma(t[i + 2].y, w[i + 2], a2.y);
        a3.x = fma(t[i + 3].x, w[i + 3], a3.x);
        a3.y = fma(t[i + 3].y, w[i + 3], a3.y);
      }
    }
    for (; r < R; r += RG) {
      const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * ld);
      const double v0 = v[r];
      a0.x = fma(t0.x, v0, a0.x);
      a0.y = fma(t0.y, v0, a0.y);
    }
  }
  const double sx = (a0.x + a1.x) + (a2.x + a3.x);
  const double sy = (a0.y + a1.y) + (a2.y + a3.y);
  __syncthreads();
  if (rg < RG) {
    red[rg * 2 * CP + 2 * cp] = sx;
    red[rg * 2 * CP + 2 * cp + 1] = sy;
  }
  __syncthreads();
  for (int c = tid; c < C; c += NT) {
    double s = 0.0;
    for (int q = 0; q < RG; ++q) s += red[q * 2 * CP + c];
    epi(c, s);
  }
}

__global__ void __launch_bounds__(NT, 1) k(int which, int R, int ld, int C, int reps, long long* out, double* sink) {
  extern __shared__ __align__(128) double sm[];
  double* T = sm;
  double* v = sm + 2 * R * ld + 64;
  double* o = v + 512;
  double* red = o + 512;
  for (int i = threadIdx.x; i < 2 * R * ld; i += NT) T[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 512; i += NT) v[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (which == 0) {
      rowdot2<NT>(T, ld, R, C, v, [&](int r, double a) { o[r] += a; });
    } else if (which == 1) {
      rowdot2x<NT>(T, ld, R, C, v, [&](int r, double a) { o[r] += a; });
    } else if (which == 3) {
      if (C == 114)
        rowdot_ct<8, 8>(T, ld, R, C, v, [&](int r, double a) { o[r] += a; });
      else
        rowdot_ct<16, 7>(T, ld, R, C, v, [&](int r, double a) { o[r] += a; });
    } else if (which == 9) {
      if (threadIdx.x < R) o[threadIdx.x] += 1.0;
    } else if (which == 8) {
      rowdot_warp<NT>(T, ld, R, C, v, [&](int r, double a) { o[r] += a; });
    } else if (which >= 5) {
      auto e = [&](int r, double a) { o[r] += a; };
      if (C == 114) {
        if (which == 5) rowdot2u_l<NT, 8, 4>(T, ld, R, C, v, e);
        if (which == 6) rowdot2u_l<NT, 8, 6>(T, ld, R, C, v, e);
        if (which == 7) rowdot2u_l<NT, 8, 8>(T, ld, R, C, v, e);
      } else {
        if (which == 5) rowdot2u_l<NT, 16, 4>(T, ld, R, C, v, e);
        if (which == 6) rowdot2u_l<NT, 16, 6>(T, ld, R, C, v, e);
        if (which == 7) rowdot2u_l<NT, 16, 7>(T, ld, R, C, v, e);
      }
    } else if (which == 4) {
      colsum_u8(T, ld, 2 * R, C, v, red, [&](int c, double a) { o[c] += a; });
    } else {
      colsum2h<NT>(
          T, T + R * ld, ld, 2 * R, R, C, v, red, []() {}, []() {}, [&](int c, double a) { o[c] += a; });
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
  sink[blockIdx.x] = o[threadIdx.x & 63];
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 8 * 1024);
  cudaMalloc(&s, 8 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  struct Shape {
    const char* nm;
    int R, ld, C;
  } shapes[] = {{"row group half (100x114)", 100, 114, 114},
                {"row group half, pitch 120", 100, 120, 114},
                {"col group half (63x200)", 63, 200, 200}};
  const char* wn[] = {"rowdot2", "rowdot2x", "colsum2h (both halves)", "rowdot_ct (unrolled)", "colsum_u8 (both halves)", "rowdot2u Q=4", "rowdot2u Q=6", "rowdot2u Q=8/7", "rowdot_warp", "empty (epilogue only)"};
  for (auto& sh : shapes) {
    for (int w = 0; w < 10; ++w) {
      const size_t smem = (2 * (size_t)sh.R * sh.ld + 64 + 512 + 512 + 1024) * 8;
      k<<<148, NT, smem>>>(w, sh.R, sh.ld, sh.C, 200, d, s);
      long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double bytes = (w == 2 || w == 4 ? 2.0 : 1.0) * sh.R * sh.C * 8;
      printf("%-28s %-24s %6lld cycles  %.3f us  %.1f B/clk  %s\n", sh.nm, wn[w], h, h / 1965.0, bytes / h,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

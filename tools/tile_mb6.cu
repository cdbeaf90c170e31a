// tile_mb6.cu — "warp owns rows, lanes own column pairs" tile products
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;

// out[r] = Σ_c T[r][c] v[c]: lanes hold their v pairs in registers; a warp
// does two rows at a time; xor-butterfly per row.
template <int NT, typename Epi>
__device__ __forceinline__ void rowdot_w(const double* __restrict__ T, int ld, int R, int C,
                                         const double* __restrict__ v, Epi epi) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int CPf = C >> 1;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  double2 vr[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) vr[j] = (lane + 32 * j < CPf) ? v2[lane + 32 * j] : make_double2(0.0, 0.0);
  const double vt = (C & 1) ? v[C - 1] : 0.0;
  const int tail_lane = CPf & 31;  // lane that owns the odd last column
  for (int r = warp; r < R; r += 2 * NW) {
    const int r2 = r + NW;
    const double2* row0 = reinterpret_cast<const double2*>(T + (size_t)r * ld);
    const double2* row1 = reinterpret_cast<const double2*>(T + (size_t)(r2 < R ? r2 : r) * ld);
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = lane + 32 * j;
      if (q < CPf) {
        const double2 t0 = row0[q], t1 = row1[q];
        a0 = fma(t0.x, vr[j].x, a0);
        a1 = fma(t0.y, vr[j].y, a1);
        b0 = fma(t1.x, vr[j].x, b0);
        b1 = fma(t1.y, vr[j].y, b1);
      }
    }
    if ((C & 1) && lane == tail_lane) {
      a0 = fma(T[(size_t)r * ld + C - 1], vt, a0);
      b0 = fma(T[(size_t)(r2 < R ? r2 : r) * ld + C - 1], vt, b0);
    }
    double a = a0 + a1, b = b0 + b1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    if (lane == 0) {
      epi(r, a);
      if (r2 < R) epi(r2, b);
    }
  }
}

// out[c] = Σ_r T[r][c] v[r]: lanes own column pairs (≤ 4 per lane), warps
// own rows; warp partials reduced in smem (two-stage, fixed order).
template <int NT, typename Epi>
__device__ __forceinline__ void colsum_w(const double* __restrict__ T, int ld, int R, int C,
                                         const double* __restrict__ v, double* red, Epi epi) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int CP = (C + 1) >> 1;
  double2 acc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j] = make_double2(0.0, 0.0);
  for (int r = warp; r < R; r += NW) {
    const double vr = v[r];
    const double2* row = reinterpret_cast<const double2*>(T + (size_t)r * ld);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = lane + 32 * j;
      if (q < CP) {
        const double2 t = row[q];
        acc[j].x = fma(t.x, vr, acc[j].x);
        acc[j].y = fma(t.y, vr, acc[j].y);
      }
    }
  }
  // warps [NW/2, NW) store, warps [0, NW/2) add theirs, then NW/2 partials per column
  constexpr int H = NW / 2;
  const int C2 = 2 * CP;
  if (warp >= H) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = lane + 32 * j;
      if (q < CP) reinterpret_cast<double2*>(red + (size_t)(warp - H) * C2)[q] = acc[j];
    }
  }
  __syncthreads();
  if (warp < H) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = lane + 32 * j;
      if (q < CP) {
        double2* p = reinterpret_cast<double2*>(red + (size_t)warp * C2) + q;
        const double2 o = *p;
        *p = make_double2(acc[j].x + o.x, acc[j].y + o.y);
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += NT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < H; ++w) s += red[(size_t)w * C2 + c];
    epi(c, s);
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k(int R, int C, int ld, int which, int reps, long long* out, double* sink) {
  extern __shared__ __align__(128) double sm[];
  double* T = sm; double* v = T + (size_t)R * ld + 16; double* red = v + 512; double* o = red + 8 * 256 + 64;
  for (int i = threadIdx.x; i < R * ld; i += NT) T[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 512; i += NT) v[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (which == 0) colsum_w<NT>(T, ld, R, C, v, red, [&](int c, double a) { o[c] = a; });
    else rowdot_w<NT>(T, ld, R, C, v, [&](int r, double a) { o[r] = a; });
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[blockIdx.x] = (t1 - t0) / reps; sink[blockIdx.x] = o[1]; }
}
template <int NT> void run(int R, int C, int ld, const char* nm) {
  long long* d; double* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 8 * 1024);
  cudaFuncSetAttribute(k<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  for (int w = 0; w < 2; ++w) {
    size_t smem = ((size_t)R * ld + 16 + 512 + 8 * 256 + 64 + 512) * 8;
    k<NT><<<148, NT, smem>>>(R, C, ld, w, 100, d, s);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("NT=%d %-16s R=%3d C=%3d ld=%3d %-7s %6lld cycles (%.1f B/clk) %s\n", NT, nm, R, C, ld, w == 0 ? "colsum" : "rowdot", h, (double)R * C * 8 / h, cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  run<256>(125, 200, 200, "split col tile"); run<512>(125, 200, 200, "split col tile");
  run<256>(200, 114, 114, "split row tile"); run<512>(200, 114, 114, "split row tile");
  run<256>(200, 114, 116, "row tile ld116"); run<512>(200, 114, 116, "row tile ld116");
  run<256>(28, 200, 200, "fused col tile"); run<256>(200, 68, 70, "fused row tile");
  return 0;
}

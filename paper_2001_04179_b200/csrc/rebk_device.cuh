// rebk_device.cuh — device helpers shared by the REBK kernels (sm_100a):
// grid barrier, mbarrier / bulk-copy / TMA PTX wrappers, tile products.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include "rebk_internal.h"

namespace rebk {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
    unsigned long long v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// non-blocking test of a phase (try_wait may suspend the thread for a while)
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ loaders
struct LdShared {
  static __device__ __forceinline__ double ld(const double* p) { return *p; }
};
struct LdNC {  // immutable A: read-only path
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
};
struct LdCG {  // state written by other CTAs during this launch: L2 only
  static __device__ __forceinline__ double ld(const double* p) { return __ldcg(p); }
};

__device__ __forceinline__ int pow2floor(int v) {
  int p = 1;
  while (p * 2 <= v) p *= 2;
  return p;
}

// out[c] = Σ_{r<R} T[r*ld + c] · v[r]  (c < C), handed to epi(c, value).
// The thread layout depends on (R, C) only, so staged and unstaged tiles give
// identical bits.
template <typename TA, typename TV, typename Epi>
__device__ __forceinline__ void tile_colsum(const double* __restrict__ T, int64_t ld, int R, int C,
                                            const double* __restrict__ v, double* red, Epi epi) {
  const int tid = threadIdx.x;
  if (C <= 0) return;
  if (C >= kThreads / 2) {
    for (int c = tid; c < C; c += kThreads) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int r = 0;
      for (; r + 4 <= R; r += 4) {
        a0 = fma(TA::ld(T + (int64_t)(r + 0) * ld + c), TV::ld(v + r + 0), a0);
        a1 = fma(TA::ld(T + (int64_t)(r + 1) * ld + c), TV::ld(v + r + 1), a1);
        a2 = fma(TA::ld(T + (int64_t)(r + 2) * ld + c), TV::ld(v + r + 2), a2);
        a3 = fma(TA::ld(T + (int64_t)(r + 3) * ld + c), TV::ld(v + r + 3), a3);
      }
      for (; r < R; ++r) a0 = fma(TA::ld(T + (int64_t)r * ld + c), TV::ld(v + r), a0);
      epi(c, (a0 + a1) + (a2 + a3));
    }
  } else {
    const int RG = kThreads / C;  // >= 2 row groups
    const int c = tid % C, rg = tid / C;
    double a0 = 0.0, a1 = 0.0;
    if (rg < RG) {
      int r = rg;
      for (; r + RG < R; r += 2 * RG) {
        a0 = fma(TA::ld(T + (int64_t)r * ld + c), TV::ld(v + r), a0);
        a1 = fma(TA::ld(T + (int64_t)(r + RG) * ld + c), TV::ld(v + r + RG), a1);
      }
      if (r < R) a0 = fma(TA::ld(T + (int64_t)r * ld + c), TV::ld(v + r), a0);
    }
    __syncthreads();
    if (rg < RG) red[tid] = a0 + a1;
    __syncthreads();
    if (tid < C) {
      double s = 0.0;
      for (int q = 0; q < RG; ++q) s += red[q * C + tid];
      epi(tid, s);
    }
    __syncthreads();
  }
}

// out[r] = Σ_{c<C} T[r*ld + c] · v[c]  (r < R), handed to epi(r, value) by
// one lane per row.  L lanes per row, xor-butterfly reduction (every lane of
// the group ends with the same bits).
template <typename TA, typename TV, typename Epi>
__device__ __forceinline__ void tile_rowdot(const double* __restrict__ T, int64_t ld, int R, int C,
                                            const double* __restrict__ v, Epi epi) {
  if (R <= 0) return;
  const int tid = threadIdx.x;
  int L = pow2floor(kThreads / R);
  L = L < 2 ? 2 : (L > 32 ? 32 : L);
  const int sub = tid % L, rsub = tid / L, rows_per_pass = kThreads / L;
  for (int r0 = 0; r0 < R; r0 += rows_per_pass) {
    const int r = r0 + rsub;
    double a0 = 0.0, a1 = 0.0;
    if (r < R && C > 0) {
      const double* row = T + (int64_t)r * ld;
      int c = sub;
      for (; c + L < C; c += 2 * L) {
        a0 = fma(TA::ld(row + c), TV::ld(v + c), a0);
        a1 = fma(TA::ld(row + c + L), TV::ld(v + c + L), a1);
      }
      if (c < C) a0 = fma(TA::ld(row + c), TV::ld(v + c), a0);
    }
    double acc = a0 + a1;
    for (int off = L / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (sub == 0 && r < R) epi(r, acc);
  }
}

// Σ_{q<G} part[q]  for one warp, lane-strided then xor butterfly.
__device__ __forceinline__ double warp_sum_cg(const double* part, int G) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int q = lane; q < G; q += 32) s += __ldcg(part + q);
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// block-wide fixed-order sum (all threads must call)
template <int NT = kThreads>
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (NT / 32); ++w) s += red[w];
  __syncthreads();
  return s;
}


__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy): streams read
// once get evict_first so they do not push out data that is read again soon
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// pull a 2D box into L2 ahead of its TMA load (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch_l2_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
               : "memory");
}
// barrier among `nthreads` threads (a multiple of 32) of the CTA on hardware barrier `id` (1..15)
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// pull a contiguous byte range (16-byte aligned, a multiple of 16 bytes) into L2
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t local_smem, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem), "r"(rank));
  return r;
}
// DSMEM store that counts 8 bytes on the receiver's mbarrier (shared::cluster addresses)
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
               "l"(__double_as_longlong(v)), "r"(remote_mbar)
               : "memory");
}
// {value, seq} published as one 16-byte store; consumers poll the same word.
// Tear-proof layout (the LL idea): each 8-byte half carries the sequence in
// its high 32 bits and one half of the value in its low 32 bits.  The PTX
// memory model guarantees single-copy atomicity for aligned accesses up to 8
// bytes only (a wider access may be observed as its 8-byte pieces), so the
// reader accepts the word only when BOTH halves show the expected sequence:
// a torn read (one half old, one half new) is retried, never consumed.
__device__ __forceinline__ void st_ll(LLWord* w, double v, unsigned long long seq) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned long long s32 = (seq & 0xffffffffull) << 32;
  const unsigned long long h0 = s32 | (bits & 0xffffffffull), h1 = s32 | (bits >> 32);
  asm volatile("{\n\t.reg .b128 t;\n\tmov.b128 t, {%1, %2};\n\tst.relaxed.gpu.global.b128 [%0], t;\n\t}" ::"l"(w),
               "l"(h0), "l"(h1)
               : "memory");
}
__device__ __forceinline__ double poll_ll(const LLWord* w, unsigned long long seq) {
  const unsigned long long s32 = seq & 0xffffffffull;
  unsigned long long h0, h1;
  do {
    asm volatile("{\n\t.reg .b128 t;\n\tld.relaxed.gpu.global.b128 t, [%2];\n\tmov.b128 {%0, %1}, t;\n\t}"
                 : "=l"(h0), "=l"(h1)
                 : "l"(w)
                 : "memory");
  } while ((h0 >> 32) != s32 || (h1 >> 32) != s32);
  return __longlong_as_double((long long)((h1 << 32) | (h0 & 0xffffffffull)));
}

// ---- shared-memory tile products of the fast path ---------------------------
// out[c] = Σ_{r<R} T[r*ld + c] · v[r] for c < C, T in shared memory (ld even,
// rows 16-byte aligned).  Threads own column pairs; RG row groups, four
// independent chains per thread; row-group partials summed in fixed order.
template <int NT = kThreads, typename Epi>
__device__ __forceinline__ void colsum2(const double* __restrict__ T, int ld, int R, int C,
                                        const double* __restrict__ v, double* red, Epi epi) {
  const int tid = threadIdx.x;
  if (C <= 0) return;
  const int CP = (C + 1) >> 1;
  int RG = NT / CP;
  if (RG > R) RG = R > 0 ? R : 1;
  const int cp = tid % CP, rg = tid / CP;
  double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
  if (rg < RG) {
    const double* col = T + 2 * cp;
    int r = rg;
    for (; r + 3 * RG < R; r += 4 * RG) {
      const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * ld);
      const double2 t1 = *reinterpret_cast<const double2*>(col + (size_t)(r + RG) * ld);
      const double2 t2 = *reinterpret_cast<const double2*>(col + (size_t)(r + 2 * RG) * ld);
      const double2 t3 = *reinterpret_cast<const double2*>(col + (size_t)(r + 3 * RG) * ld);
      const double v0 = v[r], v1 = v[r + RG], v2 = v[r + 2 * RG], v3 = v[r + 3 * RG];
      a0.x = fma(t0.x, v0, a0.x);
      a0.y = fma(t0.y, v0, a0.y);
      a1.x = fma(t1.x, v1, a1.x);
      a1.y = fma(t1.y, v1, a1.y);
      a2.x = fma(t2.x, v2, a2.x);
      a2.y = fma(t2.y, v2, a2.y);
      a3.x = fma(t3.x, v3, a3.x);
      a3.y = fma(t3.y, v3, a3.y);
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
  if (RG == 1) {
    if (rg < 1) {
      epi(2 * cp, sx);
      if (2 * cp + 1 < C) epi(2 * cp + 1, sy);
    }
    __syncthreads();
    return;
  }
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
  __syncthreads();
}

// colsum2 over a tile that arrives in two row halves (rows [0, h) at T0,
// rows [h, R) at T1, same pitch ld): rows [0, h) are summed,
// then every thread calls mid() (e.g. wait for the second half, or release
// the first half's buffer), rows [h, R) are summed, every thread calls end()
// (the tile is no longer read after it; EndSyncs: end() is a block barrier),
// then the fixed-order reduction and epi(c, sum) run as in colsum2.
template <int NT, bool EndSyncs = false, typename Mid, typename End, typename Epi>
__device__ __forceinline__ void colsum2h(const double* __restrict__ T0, const double* __restrict__ T1, int ld, int R,
                                         int h, int C,
                                         const double* __restrict__ v, double* red, Mid mid, End end, Epi epi) {
  const int tid = threadIdx.x;
  if (C <= 0) {
    mid();
    end();
    return;
  }
  const int CP = (C + 1) >> 1;
  int RG = NT / CP;
  if (RG > R) RG = R > 0 ? R : 1;
  const int cp = tid % CP, rg = tid / CP;
  double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
  auto rows = [&](const double* col, const double* vv, int r, int r1) {
    for (; r + 3 * RG < r1; r += 4 * RG) {
      const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * ld);
      const double2 t1 = *reinterpret_cast<const double2*>(col + (size_t)(r + RG) * ld);
      const double2 t2 = *reinterpret_cast<const double2*>(col + (size_t)(r + 2 * RG) * ld);
      const double2 t3 = *reinterpret_cast<const double2*>(col + (size_t)(r + 3 * RG) * ld);
      const double v0 = vv[r], v1 = vv[r + RG], v2 = vv[r + 2 * RG], v3 = vv[r + 3 * RG];
      a0.x = fma(t0.x, v0, a0.x);
      a0.y = fma(t0.y, v0, a0.y);
      a1.x = fma(t1.x, v1, a1.x);
      a1.y = fma(t1.y, v1, a1.y);
      a2.x = fma(t2.x, v2, a2.x);
      a2.y = fma(t2.y, v2, a2.y);
      a3.x = fma(t3.x, v3, a3.x);
      a3.y = fma(t3.y, v3, a3.y);
    }
    for (; r < r1; r += RG) {
      const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * ld);
      const double v0 = vv[r];
      a0.x = fma(t0.x, v0, a0.x);
      a0.y = fma(t0.y, v0, a0.y);
    }
  };
  if (h > R) h = R;
  if (rg < RG) rows(T0 + 2 * cp, v, rg, h);
  mid();
  if (rg < RG) rows(T1 + 2 * cp, v + h, rg, R - h);
  end();
  const double sx = (a0.x + a1.x) + (a2.x + a3.x);
  const double sy = (a0.y + a1.y) + (a2.y + a3.y);
  if (RG == 1) {
    if (rg < 1) {
      epi(2 * cp, sx);
      if (2 * cp + 1 < C) epi(2 * cp + 1, sy);
    }
    __syncthreads();
    return;
  }
  if (!EndSyncs) __syncthreads();  // end() may already be a block barrier
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
  __syncthreads();
}

// rowdot2 with two rows per thread (r and r + NT/L) in one pass: twice the
// loads in flight per thread and each v pair read once for both rows.  The
// second row's loads are predicated off past R.
template <int NT, typename Epi>
__device__ __forceinline__ void rowdot2x(const double* __restrict__ T, int ld, int R, int C,
                                         const double* __restrict__ v, Epi epi) {
  if (R <= 0) return;
  const int tid = threadIdx.x;
  const int CPf = C >> 1;
  int L = pow2floor((2 * NT) / R);
  const int lmax = CPf >= 1 ? pow2floor(CPf) : 1;
  L = L > 32 ? 32 : L;
  L = L > lmax ? lmax : L;
  if (L < 8) {  // bank rule of rowdot2
    const int pm = (ld * 8) & 127;
    const bool clean = pm % (16 * L) == 0 && ((pm / (16 * L)) & 1);
    if (!clean) L = lmax < 8 ? lmax : 8;
  }
  const int sub = tid % L, rsub = tid / L, rpp = NT / L;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  const double2 z2 = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < R; r0 += 2 * rpp) {
    const int ra = r0 + rsub, rb = ra + rpp;
    const bool hb = rb < R;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
    if (ra < R) {
      const double2* rowa = reinterpret_cast<const double2*>(T + (size_t)ra * ld);
      const double2* rowb = reinterpret_cast<const double2*>(T + (size_t)(hb ? rb : ra) * ld);
      int q = sub;
      for (; q + L < CPf; q += 2 * L) {
        const double2 w0 = v2[q], w1 = v2[q + L];
        const double2 s0 = rowa[q], s1 = rowa[q + L];
        const double2 t0 = hb ? rowb[q] : z2, t1 = hb ? rowb[q + L] : z2;
        a0 = fma(s0.x, w0.x, a0);
        a1 = fma(s0.y, w0.y, a1);
        a2 = fma(s1.x, w1.x, a2);
        a3 = fma(s1.y, w1.y, a3);
        b0 = fma(t0.x, w0.x, b0);
        b1 = fma(t0.y, w0.y, b1);
        b2 = fma(t1.x, w1.x, b2);
        b3 = fma(t1.y, w1.y, b3);
      }
      if (q < CPf) {
        const double2 w0 = v2[q];
        const double2 s0 = rowa[q];
        const double2 t0 = hb ? rowb[q] : z2;
        a0 = fma(s0.x, w0.x, a0);
        a1 = fma(s0.y, w0.y, a1);
        b0 = fma(t0.x, w0.x, b0);
        b1 = fma(t0.y, w0.y, b1);
      }
      if ((C & 1) && sub == (CPf % L)) {
        a2 = fma(T[(size_t)ra * ld + C - 1], v[C - 1], a2);
        if (hb) b2 = fma(T[(size_t)rb * ld + C - 1], v[C - 1], b2);
      }
    }
    double acc = (a0 + a1) + (a2 + a3), bcc = (b0 + b1) + (b2 + b3);
    for (int off = L / 2; off > 0; off >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, off);
      bcc += __shfl_xor_sync(0xffffffffu, bcc, off);
    }
    if (sub == 0 && ra < R) epi(ra, acc);
    if (sub == 0 && hb) epi(rb, bcc);
  }
}

// rowdot2x with the lane count L fixed at compile time and the pair loop
// unrolled in chunks of Q pairs per lane: all 3Q loads of a chunk (Q v pairs,
// Q pairs of each of the two rows) are issued before the first FMA.
#ifndef REBK_ROWDOT_Q
#define REBK_ROWDOT_Q 4
#endif
template <int NT, int L, int Q = REBK_ROWDOT_Q, typename Epi>
__device__ __forceinline__ void rowdot2u_l(const double* __restrict__ T, int ld, int R, int C,
                                           const double* __restrict__ v, Epi epi) {
  constexpr int rpp = NT / L;
  const int tid = threadIdx.x;
  const int CPf = C >> 1;
  const int sub = tid % L, rsub = tid / L;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  const double2 z2 = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < R; r0 += 2 * rpp) {
    const int ra = r0 + rsub, rb = ra + rpp;
    const bool ha = ra < R, hb = rb < R;
    const double2* rowa = reinterpret_cast<const double2*>(T + (size_t)(ha ? ra : 0) * ld);
    const double2* rowb = reinterpret_cast<const double2*>(T + (size_t)(hb ? rb : 0) * ld);
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    for (int q0 = sub; q0 < CPf; q0 += Q * L) {
      double2 w[Q], s[Q], t[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const int q = q0 + i * L;
        const bool in = q < CPf;
        w[i] = in ? v2[q] : z2;
        s[i] = (in && ha) ? rowa[q] : z2;
        t[i] = (in && hb) ? rowb[q] : z2;
      }
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        a0 = fma(s[i].x, w[i].x, a0);
        a1 = fma(s[i].y, w[i].y, a1);
        b0 = fma(t[i].x, w[i].x, b0);
        b1 = fma(t[i].y, w[i].y, b1);
      }
    }
    if ((C & 1) && sub == (CPf % L)) {
      if (ha) a0 = fma(T[(size_t)ra * ld + C - 1], v[C - 1], a0);
      if (hb) b0 = fma(T[(size_t)rb * ld + C - 1], v[C - 1], b0);
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

// out[r] = Σ_{c<C} T[r*ld + c] · v[c] for r < R with whole warps per row:
// lane l owns the column pairs l + 32i (i < PB), so its slice of v stays in
// registers for the whole call; warp w owns rows w, w + NW, ... and keeps the
// loads of 4 rows x PB pairs in flight before the FMAs; one 5-level xor
// butterfly per row.  Every tile load is a contiguous 512-byte warp read
// (4 wavefronts, no bank conflicts for any pitch) and v costs no wavefronts.
// Needs C <= 64 * PB.
template <int NT, int PB, typename Epi>
__device__ __forceinline__ void rowdot_w(const double* __restrict__ T, int ld, int R, int C,
                                         const double* __restrict__ v, Epi epi) {
  constexpr int NW = NT / 32, RB = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int CPf = C >> 1;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  const double2 z2 = make_double2(0.0, 0.0);
  double2 w[PB];
#pragma unroll
  for (int i = 0; i < PB; ++i) w[i] = lane + 32 * i < CPf ? v2[lane + 32 * i] : z2;
  const bool odd = (C & 1) && lane == 0;
  const double vlast = odd ? v[C - 1] : 0.0;
  for (int r0 = warp; r0 < R; r0 += RB * NW) {
    double2 t[RB][PB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const int r = r0 + j * NW;
      const double2* row = reinterpret_cast<const double2*>(T + (size_t)(r < R ? r : 0) * ld);
#pragma unroll
      for (int i = 0; i < PB; ++i) t[j][i] = (r < R && lane + 32 * i < CPf) ? row[lane + 32 * i] : z2;
    }
    double acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        a0 = fma(t[j][i].x, w[i].x, a0);
        a1 = fma(t[j][i].y, w[i].y, a1);
      }
      const int r = r0 + j * NW;
      if (odd && r < R) a0 = fma(T[(size_t)r * ld + C - 1], vlast, a0);
      acc[j] = a0 + a1;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int j = 0; j < RB; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < RB; ++j)
        if (r0 + j * NW < R) epi(r0 + j * NW, acc[j]);
  }
}

template <int NT, typename Epi>
__device__ __forceinline__ void rowdot_warp(const double* __restrict__ T, int ld, int R, int C,
                                            const double* __restrict__ v, Epi epi) {
  if (R <= 0) return;
  switch (((C >> 1) + 31) >> 5) {
    case 0:
    case 1: rowdot_w<NT, 1>(T, ld, R, C, v, epi); break;
    case 2: rowdot_w<NT, 2>(T, ld, R, C, v, epi); break;
    case 3: rowdot_w<NT, 3>(T, ld, R, C, v, epi); break;
    case 4: rowdot_w<NT, 4>(T, ld, R, C, v, epi); break;
    default: rowdot2x<NT>(T, ld, R, C, v, epi); break;  // wider than 256 columns
  }
}

// Lane count as in rowdot2x (two rows per thread, bank rule), dispatched to
// the compile-time kernel (L >= 8: tiles of at most 2*NT/8 rows).
template <int NT, typename Epi>
__device__ __forceinline__ void rowdot2u(const double* __restrict__ T, int ld, int R, int C,
                                         const double* __restrict__ v, Epi epi) {
  if (R <= 0) return;
  const int CPf = C >> 1;
  int L = pow2floor((2 * NT) / R);
  const int lmax = CPf >= 1 ? pow2floor(CPf) : 1;
  L = L > 32 ? 32 : L;
  L = L > lmax ? lmax : L;
  if (L < 8) {
    const int pm = (ld * 8) & 127;
    const bool clean = pm % (16 * L) == 0 && ((pm / (16 * L)) & 1);
    if (!clean) L = lmax < 8 ? lmax : 8;
  }
  switch (L) {
    // Q: one chunk covers 64 (L=8) / 112 (L=16) / 128 (L=32) column pairs
    // Q = 4 pairs per lane per chunk: 24 loads in flight per thread without
    // spilling inside the 128-register budget of the 512-thread split kernel
    case 32: rowdot2u_l<NT, 32, REBK_ROWDOT_Q>(T, ld, R, C, v, epi); break;
    case 16: rowdot2u_l<NT, 16, REBK_ROWDOT_Q>(T, ld, R, C, v, epi); break;
    case 8: rowdot2u_l<NT, 8, REBK_ROWDOT_Q>(T, ld, R, C, v, epi); break;
    default: rowdot2x<NT>(T, ld, R, C, v, epi); break;  // tall or narrow tiles
  }
}

// out[r] = Σ_{c<C} T[r*ld + c] · v[c] for r < R.  L lanes per row read
// 16-byte pairs; xor butterfly inside the lane group.  An odd trailing column
// is handled by one lane so v needs no padding.
template <int NT = kThreads, typename Epi>
__device__ __forceinline__ void rowdot2(const double* __restrict__ T, int ld, int R, int C,
                                        const double* __restrict__ v, Epi epi) {
  if (R <= 0) return;
  const int tid = threadIdx.x;
  const int CPf = C >> 1;  // full pairs
  int L = pow2floor(NT / R);
  const int lmax = CPf >= 1 ? pow2floor(CPf) : 1;
  L = L > 32 ? 32 : L;
  L = L > lmax ? lmax : L;
  if (L < 8) {
    // a quarter-warp (8 lanes, one 128-byte wavefront) covers 8/L rows of
    // 16L bytes each; they hit distinct banks only if the row pitch is an odd
    // multiple of 16L bytes mod 128.  Otherwise give each row 8 lanes (one
    // row per quarter-warp: conflict-free for any pitch).
    const int pm = (ld * 8) & 127;
    const bool clean = pm % (16 * L) == 0 && ((pm / (16 * L)) & 1);
    if (!clean) L = lmax < 8 ? lmax : 8;
  }
  const int sub = tid % L, rsub = tid / L, rpp = NT / L;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  for (int r0 = 0; r0 < R; r0 += rpp) {
    const int r = r0 + rsub;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    if (r < R) {
      const double2* row = reinterpret_cast<const double2*>(T + (size_t)r * ld);
      int q = sub;
      for (; q + L < CPf; q += 2 * L) {
        const double2 t0 = row[q], t1 = row[q + L];
        const double2 w0 = v2[q], w1 = v2[q + L];
        c0 = fma(t0.x, w0.x, c0);
        c1 = fma(t0.y, w0.y, c1);
        c2 = fma(t1.x, w1.x, c2);
        c3 = fma(t1.y, w1.y, c3);
      }
      if (q < CPf) {
        const double2 t0 = row[q], w0 = v2[q];
        c0 = fma(t0.x, w0.x, c0);
        c1 = fma(t0.y, w0.y, c1);
      }
      if ((C & 1) && sub == (CPf % L)) c2 = fma(T[(size_t)r * ld + C - 1], v[C - 1], c2);
    }
    double acc = (c0 + c1) + (c2 + c3);
    for (int off = L / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (sub == 0 && r < R) epi(r, acc);
  }
}

// Cluster barrier with release/acquire at cluster scope only.  (cg's
// cluster.sync() also emits a GPU-scope MEMBAR, which is not needed for DSMEM
// traffic and costs a full drain of outstanding global stores.)
__device__ __forceinline__ void cluster_sync_rel_acq() {
#ifdef REBK_CG_CLUSTER_SYNC
  cooperative_groups::this_cluster().sync();
#else
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#endif
}

}  // namespace rebk

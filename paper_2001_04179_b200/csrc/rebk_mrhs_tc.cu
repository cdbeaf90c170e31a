// rebk_mrhs_tc.cu — multi-RHS fp32 REBK (BASELINE config 5) on the 5th-gen
// tensor cores: hand-written tcgen05 kind::tf32 GEMMs with 3xTF32 operand
// splitting (fp32 accuracy), accumulators in TMEM.
//
// kind::tf32 takes K-major operands only, so everything is arranged for K to
// be the contiguous dimension in HBM:
//   * A (m x n, row-major) and a transposed copy At (n x m, built once per
//     context) — the column sweep reads At rows, the row sweep A rows;
//   * the iterates live transposed, Zt (R x m) and Xt (R x n), and so do the
//     small per-iteration vectors Ut (R x |J|) and Rt (R x |I|).
// The four products of step_rebk (solvers.py:283-295) are then
//   U  = A_Jᵀ Z    : D[j][c] = Σ_r At[c_lo+j][r] · Zt[c][r]     (split over r)
//   Z -= s A_J U   : D[r][c] = Σ_j A[r][c_lo+j] · Ut[c][j]     (tiles of 128 r)
//   Rr = A_I X..   : D[i][c] = Σ_k A[r_lo+i][k] · Xt[c][k]     (split over k)
//   X -= s A_Iᵀ Rr : D[k][c] = Σ_i At[k][r_lo+i] · Rt[c][i]    (tiles of 128 k)
// with c the right-hand side.  Every operand tile is one 2D TMA box of 32
// fp32 along K (128 bytes) x rows with the 128-byte swizzle, i.e. exactly the
// K-major SWIZZLE_128B UMMA layout (umma.cuh).  (A no-swizzle layout needs
// 16-byte-wide boxes, which TMA moves far too slowly.)  3xTF32:
// D += hi·hi + hi·lo + lo·hi; the raw fp32 tile serves as "hi" (the tensor
// core truncates to TF32, measured bit-identical to an explicit split) and
// the CTA computes the lo tiles in shared memory.  Partial sums of the split
// products are reduced in a fixed order, so runs replay bit for bit.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/rebk.h"
#include "rebk_device.cuh"
#include "rebk_internal.h"
#include "umma.cuh"

namespace rebk {

namespace tc {

constexpr int BK = 32;           // K per pipeline stage: one 128-byte swizzle atom (4 tf32 MMA k-steps)
constexpr int NSTAGE = 4;
constexpr int TM = 128;          // MMA M (rows per tile)
constexpr int RHS = 64;          // MMA N = number of right-hand sides

// shared memory of one stage (floats): A raw, A lo, B raw, B lo
constexpr int STAGE_FLOATS = 2 * TM * BK + 2 * RHS * BK;
constexpr size_t SMEM_BYTES = (size_t)NSTAGE * STAGE_FLOATS * 4 + 1024;  // + alignment slack

__device__ __forceinline__ float* aligned_smem(float* p) {
  return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~(uintptr_t)1023);
}

// ---- warp-specialized persistent GEMM -----------------------------------------
// 12 warps: warp 0 = TMA producer, warp 1 = MMA issuer (one lane each),
// warps 2-7 = converters (lo = x - trunc_tf32(x) into the stage's lo tiles),
// warps 8-11 = epilogue (TMEM lanes 32*(warp%4)..).  Ring of NSTAGE stages
// (raw A, lo A, raw B, lo B); two TMEM accumulators (D_hh | D_hl, 128
// columns each) so the epilogue of one tile overlaps the next tile's MMAs.
// Work list: tile j of this CTA = (row0, k-block range); MODE 0 writes split-K
// partials, MODE 1 applies Yt[c][row] -= s * D[row][c].
constexpr int NTW = 384;
constexpr int CONV0 = 2, NCONV = 6, EPI0 = 8;

struct Pipe {
  uint64_t full[NSTAGE], conv[NSTAGE], empty[NSTAGE];
  uint64_t tfull[2], tempty[2];
  uint32_t tmem;
};

struct TileJob {
  int row0;   // first operand row of the tile
  int kb0, kb1;
  int slot;   // output index: partial slice (MODE 0) / unused
};

template <int MODE>
__global__ void __launch_bounds__(NTW, 1)
    k_gemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int a_k0, int row_lo,
           int nrows, int nkb, int nslices, float s, float* __restrict__ out, int64_t ldy, int dbg) {
  extern __shared__ float smem_raw[];
  float* smem = aligned_smem(smem_raw);
  __shared__ Pipe P;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) umma::tmem_alloc<256>(&P.tmem);
  if (tid == 32) {
    for (int q = 0; q < NSTAGE; ++q) {
      mbar_init(&P.full[q], 1);
      mbar_init(&P.conv[q], NCONV);
      mbar_init(&P.empty[q], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&P.tfull[b], 1);
      mbar_init(&P.tempty[b], 4);
    }
    fence_mbar_init();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = P.tmem;

  // this CTA's tiles: MODE 0 -> one (row tile, K slice); MODE 1 -> row tiles
  // blockIdx.x, +gridDim.x, ... with the whole K range
  const int ntiles_total = (nrows + TM - 1) / TM;
  const int ntiles_part = (nrows + TM - 1) / TM;  // MODE 0: row tiles, all for this CTA's K slice
  auto job = [&](int j, TileJob& J) -> bool {
    if (MODE == 0) {
      if (j >= ntiles_part) return false;
      const int t = j, q = blockIdx.x;
      J.row0 = row_lo + t * TM;
      J.kb0 = (int)((int64_t)nkb * q / nslices);
      J.kb1 = (int)((int64_t)nkb * (q + 1) / nslices);
      J.slot = q;
      return true;
    }
    const int tau = blockIdx.x + j * gridDim.x;
    if (tau >= ntiles_total) return false;
    J.row0 = tau * TM;
    J.kb0 = 0;
    J.kb1 = nkb;
    J.slot = tau;
    return true;
  };
  auto a_raw = [&](int q) { return smem + (size_t)q * STAGE_FLOATS; };
  auto a_lo = [&](int q) { return smem + (size_t)q * STAGE_FLOATS + TM * BK; };
  auto b_raw = [&](int q) { return smem + (size_t)q * STAGE_FLOATS + 2 * TM * BK; };
  auto b_lo = [&](int q) { return smem + (size_t)q * STAGE_FLOATS + 2 * TM * BK + RHS * BK; };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      uint32_t ph = 0;
      int it = 0;
      TileJob J;
      // pull every block of this CTA into L2 first: the DRAM then sees whole
      // row segments at once, and the ring's TMA loads hit L2
      if (dbg & 4)
        for (int j = 0; job(j, J); ++j)
          for (int kb = J.kb0; kb < J.kb1; ++kb) {
            tma_prefetch_l2_2d(&ma, a_k0 + kb * BK, J.row0);
            if (j == 0) tma_prefetch_l2_2d(&mb, kb * BK, 0);
          }
      for (int j = 0; job(j, J); ++j)
        for (int kb = J.kb0; kb < J.kb1; ++kb, ++it) {
          const int q = it % NSTAGE;
          if (it >= NSTAGE) {
            mbar_wait(&P.empty[q], (ph >> q) & 1u);
            ph ^= 1u << q;
          }
          mbar_arrive_expect_tx(&P.full[q], (TM + RHS) * BK * 4);
          tma_load_2d(a_raw(q), &ma, a_k0 + kb * BK, J.row0, &P.full[q]);
          tma_load_2d(b_raw(q), &mb, kb * BK, 0, &P.full[q]);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      const uint32_t idesc = umma::idesc_tf32(TM, RHS);
      uint32_t phc = 0, pht = 0;
      int it = 0;
      TileJob J;
      for (int j = 0; job(j, J); ++j) {
        const int b = j & 1;
        if (j >= 2) {  // accumulator b is free once the epilogue of tile j-2 has read it
          mbar_wait(&P.tempty[b], (pht >> b) & 1u);
          pht ^= 1u << b;
        }
        const uint32_t dh = tmem + b * 128, dl = dh + RHS;
        for (int kb = J.kb0; kb < J.kb1; ++kb, ++it) {
          const int q = it % NSTAGE;
          mbar_wait(&P.conv[q], (phc >> q) & 1u);
          phc ^= 1u << q;
          umma::fence_after_sync();
          for (int ks = 0; ks < ((dbg & 2) ? 0 : BK / 8); ++ks) {
            const uint64_t ah = umma::make_desc_sw128(smem_u32(a_raw(q)) + 32 * ks);
            const uint64_t al = umma::make_desc_sw128(smem_u32(a_lo(q)) + 32 * ks);
            const uint64_t bh = umma::make_desc_sw128(smem_u32(b_raw(q)) + 32 * ks);
            const uint64_t bl = umma::make_desc_sw128(smem_u32(b_lo(q)) + 32 * ks);
            const bool acc = kb > J.kb0 || ks > 0;
            umma::mma_tf32(dh, ah, bh, idesc, acc);
            umma::mma_tf32(dl, ah, bl, idesc, acc);
            umma::mma_tf32(dh, al, bh, idesc, true);
          }
          umma::commit(&P.empty[q]);
        }
        umma::commit(&P.tfull[b]);  // (an empty K range leaves D untouched; see the epilogue)
      }
    }
  } else if (warp < EPI0) {  // ---- converters
    const int ct = tid - CONV0 * 32;
    uint32_t phf = 0;
    int it = 0;
    TileJob J;
    for (int j = 0; job(j, J); ++j)
      for (int kb = J.kb0; kb < J.kb1; ++kb, ++it) {
        const int q = it % NSTAGE;
        mbar_wait(&P.full[q], (phf >> q) & 1u);
        phf ^= 1u << q;
        constexpr int A4 = TM * BK / 4, B4 = RHS * BK / 4;
        for (int e = ct; e < ((dbg & 1) ? 0 : A4 + B4); e += NCONV * 32) {
          const float4* src = e < A4 ? reinterpret_cast<const float4*>(a_raw(q)) + e
                                     : reinterpret_cast<const float4*>(b_raw(q)) + (e - A4);
          float4* dst = e < A4 ? reinterpret_cast<float4*>(a_lo(q)) + e : reinterpret_cast<float4*>(b_lo(q)) + (e - A4);
          const float4 v = *src;
          float4 l;
          float h;
          umma::split_tf32(v.x, h, l.x);
          umma::split_tf32(v.y, h, l.y);
          umma::split_tf32(v.z, h, l.z);
          umma::split_tf32(v.w, h, l.w);
          *dst = l;
        }
        fence_proxy_async();  // this thread's generic smem writes -> async proxy
        __syncwarp();
        if (lane == 0) mbar_arrive(&P.conv[q]);
      }
  } else {  // ---- epilogue
    uint32_t pht = 0;
    TileJob J;
    const int rlane = (warp & 3) * 32;
    for (int j = 0; job(j, J); ++j) {
      const int b = j & 1;
      mbar_wait(&P.tfull[b], (pht >> b) & 1u);
      pht ^= 1u << b;
      umma::fence_after_sync();
      const uint32_t base = tmem + ((uint32_t)rlane << 16) + b * 128;
      const int row = rlane + lane;
      const bool any = J.kb1 > J.kb0;
      for (int c0 = 0; c0 < RHS; c0 += 16) {
        float h[16], l[16];
        umma::tmem_ld16(base + c0, h);
        umma::tmem_ld16(base + RHS + c0, l);
        if (MODE == 0) {
          const int jrow = J.row0 - row_lo + row;
          if (jrow < nrows) {
            float4* dst = reinterpret_cast<float4*>(out + ((size_t)J.slot * 256 + jrow) * RHS + c0);
#pragma unroll
            for (int w = 0; w < 4; ++w)
              dst[w] = any ? make_float4(h[4 * w] + l[4 * w], h[4 * w + 1] + l[4 * w + 1], h[4 * w + 2] + l[4 * w + 2],
                                         h[4 * w + 3] + l[4 * w + 3])
                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        } else {
          const int r = J.row0 + row;
          if (r < nrows && any) {
            float y[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) y[q] = __ldcg(out + (size_t)(c0 + q) * ldy + r);
#pragma unroll
            for (int q = 0; q < 16; ++q) __stcg(out + (size_t)(c0 + q) * ldy + r, y[q] - s * (h[q] + l[q]));
          }
        }
      }
      umma::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&P.tempty[b]);
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<256>(tmem);
}

// Split-K sums, fixed order: block (row j of 256, 32 columns c) with 8 warps;
// warp g sums partials q = g, g + 8, ... for its lane's column, then lane
// c of warp 0 adds the 8 group sums in order.
__device__ __forceinline__ float sum_parts(const float* __restrict__ part, int nparts, int j, int c) {
  __shared__ float grp[8][32];
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int q = g; q < nparts; q += 8) acc += part[((size_t)q * 256 + j) * RHS + c];
  grp[g][lane] = acc;
  __syncthreads();
  float s = 0.f;
  if (g == 0)
    for (int w = 0; w < 8; ++w) s += grp[w][lane];
  return s;
}
// Ut[c][j] = Σ_q part[q][j][c] for j < nJ, zero for nJ <= j < 256 (K padding)
__global__ void __launch_bounds__(256) k_reduce_u(const float* __restrict__ part, int nparts, int nJ, int ldu,
                                                  float* __restrict__ Ut) {
  const int j = blockIdx.x, c = blockIdx.y * 32 + (threadIdx.x & 31);
  const float s = j < nJ ? sum_parts(part, nparts, j, c) : 0.f;
  if (threadIdx.x < 32) Ut[(size_t)c * ldu + j] = s;
}
// Rt[c][i] = ((Σ_q part[q][i][c]) - Bt[c][r_lo+i]) + Zt[c][r_lo+i]  (solvers.py:291-293 order)
__global__ void __launch_bounds__(256) k_reduce_r(const float* __restrict__ part, int nparts, int nI, int ldr,
                                                  const float* __restrict__ Bt, const float* __restrict__ Zt,
                                                  int64_t ldm, int r_lo, float* __restrict__ Rt) {
  const int i = blockIdx.x, c = blockIdx.y * 32 + (threadIdx.x & 31);
  float v = 0.f;
  if (i < nI) {
    v = sum_parts(part, nparts, i, c);
    if (threadIdx.x < 32) {
      v = v - Bt[(size_t)c * ldm + r_lo + i];
      if (Zt) v += Zt[(size_t)c * ldm + r_lo + i];
    }
  }
  if (threadIdx.x < 32) Rt[(size_t)c * ldr + i] = v;
}

// out[c][r] = in[r][c] for the R columns of a row-major (rows x R) array
// (columns R..63 of the transposed array stay zero), and the inverse
__global__ void k_to_t(const float* __restrict__ in, int64_t rows, int R, float* __restrict__ out, int64_t ldo) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y;
    const int c = c0 + threadIdx.x;
    t[y][threadIdx.x] = (r < rows && c < R) ? in[r * R + c] : 0.f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + threadIdx.x;
    if (r < rows) out[(size_t)(c0 + y) * ldo + r] = t[threadIdx.x][y];
  }
}
__global__ void k_from_t(const float* __restrict__ in, int64_t ldi, int64_t rows, int R, float* __restrict__ out) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + threadIdx.x;
    t[y][threadIdx.x] = r < rows ? in[(size_t)(c0 + y) * ldi + r] : 0.f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y;
    const int c = c0 + threadIdx.x;
    if (r < rows && c < R) out[r * R + c] = t[threadIdx.x][y];
  }
}
__global__ void k_transpose(const float* __restrict__ A, int64_t m, int64_t n, int64_t lda, float* __restrict__ At,
                            int64_t ldat) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y, c = c0 + threadIdx.x;
    t[y][threadIdx.x] = (r < m && c < n) ? A[r * lda + c] : 0.f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y, r = r0 + threadIdx.x;
    if (c < n && r < m) At[c * ldat + r] = t[threadIdx.x][y];
  }
}

// per-RHS ||Xt[c] - Xst[c]||^2: chunk partials (fixed order) + crossing logic
constexpr int kChk = 1024;
__global__ void k_check_part(const float* __restrict__ Xt, const float* __restrict__ Xst, int64_t n,
                             double* __restrict__ part) {
  __shared__ double red[8];
  const int c = blockIdx.y;
  const int64_t k0 = (int64_t)blockIdx.x * kChk;
  double acc = 0.0;
  for (int64_t k = k0 + threadIdx.x; k < k0 + kChk && k < n; k += blockDim.x) {
    const double d = (double)Xt[(size_t)c * n + k] - (double)Xst[(size_t)c * n + k];
    acc = fma(d, d, acc);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part[(size_t)c * gridDim.x + blockIdx.x] = s;
  }
}
__global__ void k_check_final(const double* __restrict__ part, int nchunks, int R, const double* __restrict__ tol,
                              int64_t k, int64_t* iters, double* errs_at, int32_t* n_done) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= R) return;
  double s = 0.0;
  for (int q = 0; q < nchunks; ++q) s += part[(size_t)c * nchunks + q];
  const double e = sqrt(s);
  if (iters[c] < 0 && e <= tol[c]) {
    iters[c] = k;
    errs_at[c] = e;
    atomicAdd(n_done, 1);
  }
}

// ---- persistent whole-run kernel ------------------------------------------------
// One cooperative launch runs every iteration of a chunk.  The four products
// of an iteration and the two split-K reductions are phases separated by
// grid-wide barriers (a monotonically increasing arrival counter), and the
// phases are arranged so that independent products share a phase:
//   A_k: P4(k-1)  X -= s A_Iᵀ R    (the previous iteration's x update)
//        P1(k)    U partials = A_Jᵀ Z over K slices of m
//   B_k: U = Σ partials; stop check of iteration k-1 (every CTA decides
//        redundantly from the per-tile error partials P4 wrote)
//   C_k: P2(k)    Z -= s A_J U
//        P3(k)    R partials = A_I X over K slices of n
//   D_k: R = (Σ partials - B_I) + Z_I
// (P1(k) needs Z_{k-1} only, P3(k) needs X_{k-1} only.)  Four barriers per
// iteration instead of six kernels; the run stops inside the kernel with the
// exact state of the first check at which every column has crossed, so no
// checkpoint/replay is needed.  Warp roles as in k_gemm; the converter and
// epilogue warps (320 threads) also do the reductions.
struct PkArgs {
  const Plan* plan;
  int64_t k_begin, k_end;  // iterations of this launch
  int m, n, nkb_m, nkb_n;
  int extended, checking, stride;
  int64_t max_iters;
  int ns1;           // P1 K slices (CTA pairs 2q, 2q+1 = the two 128-row halves of the column block)
  int ns3, p3_first; // P3 K slices (CTA pairs from p3_first)
  int nt2, nt4;      // 128-row tiles of the z and x updates
  int R;
  float *Zt, *Xt, *Ut, *Rt, *part1, *part3;
  const float *Bt, *Xst;
  double* errpart;        // [nt4][RHS] per-tile Σ (x - x*)^2 of a check iteration
  const double* tol;      // [R]
  int64_t* iters;         // [R] first crossing (-1: not yet)
  double* errs_at;        // [R]
  int64_t* k_final;       // iteration of the final state
  int32_t* stopped;       // set when every column has crossed
  unsigned long long* gbar;
  unsigned long long* trace;  // REBK_PK_TRACE: globaltimer stamps [iteration][CTA][8]
  int64_t trace_k0;
  int trace_n;
  unsigned long long* trace2;
  long long* trace3;  // -DPK_STAGE_TRACE: clock64 stamps [stage][8] of CTA 0 at iteration trace_k0
  int prefetch;  // L2 prefetch of the next phase's A boxes
  int dbg;       // REBK_PK_DBG experiments (8: check without the warp sums, 16: check without x* loads)
};
struct PJob {
  int kind;  // 1: P1, 2: P2, 3: P3, 4: P4
  int row0, kc0, kb0, kb1, slot, prow;
  float s;
  int check;
};
constexpr int PK_TRACE_SLOTS = 16;  // globaltimer stamps per (iteration, CTA)
constexpr int NRED = NTW - CONV0 * 32;  // threads of the reduction phases (converter + epilogue warps)

// non-aligned named barrier: callers may arrive from divergent code (e.g.
// right after one lane polled the grid barrier)
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// PK_GBAR_FENCE: 2 = __threadfence() before the release add (fence.sc),
// 1 = fence.acq_rel.gpu, 0 = the release add alone (its release semantics are
// cumulative over the CTA's writes ordered before it by the named barrier)
#ifndef PK_P4_WEIGHT_X4
#define PK_P4_WEIGHT_X4 6  // 4 x (cost of a P4 k-block in P1 stages): 6 measured best (82.9 vs 83.7 ms at 4, 8)
#endif
#ifndef PK_GBAR_FENCE
#define PK_GBAR_FENCE 0  // measured on C5: 0 98.8 ms, 1 101.4, 2 102.0 per solve
#endif
__device__ __forceinline__ void gbar_arrive(unsigned long long* g) {
#if PK_GBAR_FENCE == 2
  __threadfence();
#elif PK_GBAR_FENCE == 1
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(g) : "memory");
}
__device__ __forceinline__ void gbar_wait(const unsigned long long* g, unsigned long long target) {
  unsigned long long v;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(g) : "memory");
  } while (v < target);
}
// L2 loads of data other CTAs wrote during this launch.  __ldcg is a
// non-volatile asm without a memory clobber, so the compiler may hoist it
// above a barrier; these may not move.
__device__ __forceinline__ float ld_cg_f32(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_cg_f64(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void pk_stamp(const PkArgs& a, int64_t k, int i) {
  if (a.trace && k >= a.trace_k0 && k < a.trace_k0 + a.trace_n) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[((size_t)(k - a.trace_k0) * gridDim.x + blockIdx.x) * PK_TRACE_SLOTS + i] = t;
  }
}
// per-job stamps of CTAs 0 and 120 at iteration trace_k0 (events: 0 producer
// starts the job, 1 producer issued its last stage, 2 MMA got the first
// converted stage, 3 MMA committed the job, 4 epilogue has the accumulator,
// 5 epilogue done)
__device__ __forceinline__ void pk_jstamp(const PkArgs& a, int64_t k, int phase, int j, int ev) {
  if (a.trace && k == a.trace_k0 && (blockIdx.x == 0 || blockIdx.x == 120) && j < 4) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int sel = blockIdx.x == 0 ? 0 : 1;
    a.trace2[((sel * 2 + phase) * 4 + j) * 8 + ev] = t;
  }
}
// per-stage stamps (CTA 0, iteration trace_k0, first PK_STAGE_TRACE_N stages;
// SM clock): 0 producer saw the stage free, 1 producer issued it, 2 A
// converter saw it full, 3 A converter's TMEM stores done, 4 B converter
// done, 5 MMA thread saw it converted, 6 MMA thread committed it
constexpr int PK_STAGE_TRACE_N = 96;
#ifdef PK_STAGE_TRACE
#define PK_SC_NEXT(k, sc) if ((k) == a.trace_k0) ++(sc)
#else
#define PK_SC_NEXT(k, sc) (void)(sc)
#endif
__device__ __forceinline__ void pk_sstamp(const PkArgs& a, int64_t k, int cnt, int ev) {
#ifdef PK_STAGE_TRACE
  if (a.trace3 && blockIdx.x == 0 && k == a.trace_k0 && cnt < PK_STAGE_TRACE_N) a.trace3[cnt * 12 + ev] = clock64();
#else
  (void)a; (void)k; (void)cnt; (void)ev;
#endif
}
__device__ __forceinline__ bool pk_is_check(const PkArgs& a, int64_t k) {
  return a.checking && k >= 1 && (k % a.stride == 0 || k == a.max_iters);
}
// job j of this CTA in phase 0 (A_k) or 1 (C_k) of round k
__device__ __forceinline__ bool pk_job(const PkArgs& a, int phase, int64_t k, int j, PJob& J) {
  const int b = blockIdx.x, G = gridDim.x;
  int idx = 0;
  if (phase == 0) {
    if (k - 1 >= a.k_begin && b < a.nt4) {
      if (idx++ == j) {
        const Plan& pl = a.plan[k - 1 - a.k_begin];
        J = PJob{4, b * TM, pl.r_lo, 0, (pl.r_hi - pl.r_lo + BK - 1) / BK, b, 0, (float)pl.r_scale,
                 pk_is_check(a, k - 1) ? 1 : 0};
        return true;
      }
    }
    if (a.extended && k <= a.k_end) {
      const Plan& pl = a.plan[k - a.k_begin];
      const int q = b >> 1, h = b & 1;
      if (q < a.ns1 && h * TM < pl.c_hi - pl.c_lo && idx++ == j) {
        // pairs whose CTAs also run a P4 tile (CTAs < nt4) get kb4 fewer K
        // blocks of m, so every CTA streams about the same number of stages
        int kb4 = 0, np4 = 0;
        if (k - 1 >= a.k_begin) {
          const Plan& pp = a.plan[k - 1 - a.k_begin];
          kb4 = ((pp.r_hi - pp.r_lo + BK - 1) / BK) * PK_P4_WEIGHT_X4 / 4;  // P4 job cost in P1 stages
          np4 = (a.nt4 + 1) / 2;
        }
        const int64_t T = (int64_t)a.nkb_m + (int64_t)kb4 * np4;
        if (T - (int64_t)kb4 * a.ns1 < (int64_t)a.ns1) kb4 = 0;  // degenerate: plain even split
#ifdef PK_NO_WEIGHT
        kb4 = 0;
#endif
        const int64_t T2 = (int64_t)a.nkb_m + (int64_t)kb4 * np4;
        auto start = [&](int qq) {
          return (int)(((int64_t)qq * T2 - (int64_t)kb4 * a.ns1 * (qq < np4 ? qq : np4)) / a.ns1);
        };
        J = PJob{1, pl.c_lo + h * TM, 0, start(q), start(q + 1), q, h * TM, 0.f, 0};
        return true;
      }
    }
    return false;
  }
  const Plan& pl = a.plan[k - a.k_begin];
  int cnt2 = 0;
  if (a.extended && b < a.nt2) cnt2 = (a.nt2 - b + G - 1) / G;
  if (j < cnt2) {
    J = PJob{2, (b + j * G) * TM, pl.c_lo, 0, (pl.c_hi - pl.c_lo + BK - 1) / BK, 0, 0, (float)pl.c_scale, 0};
    return true;
  }
  idx = cnt2;
  if (b >= a.p3_first) {
    const int q = (b - a.p3_first) >> 1, h = (b - a.p3_first) & 1;
    if (q < a.ns3 && h * TM < pl.r_hi - pl.r_lo && idx == j) {
      J = PJob{3, pl.r_lo + h * TM, 0, (int)((int64_t)a.nkb_n * q / a.ns3), (int)((int64_t)a.nkb_n * (q + 1) / a.ns3), q,
               h * TM, 0.f, 0};
      return true;
    }
  }
  return false;
}

// Persistent kernel data path.  The GEMM phases are bound by the number of
// tcgen05.mma instructions (~110-130 cycles each at M = 128, K = 8, N = 64
// or 128, measured: tools/umma_ts_test.cu and the per-job trace), so each
// 8-wide k-step issues two MMAs instead of three: A_hi·[B_hi | B_lo] as one
// N = 128 MMA into the adjacent D_hh | D_hl accumulators, and A_lo·B_hi.
// A's hi and lo parts live in TMEM (the "TS" MMA form reads A from TMEM:
// converter warps 4-7 own TMEM lane quadrants 0-3 and write their rows with
// tcgen05.st), which also takes A's operand reads off shared memory.
// Rings: PK_NRAW raw stages in shared memory (A 16 KB, B 8 KB, B lo 8 KB
// written by converter warps 2-3 right behind B); PK_NA A stages in TMEM
// (hi 32 + lo 32 columns each, after the two 128-column accumulators).
#ifndef PK_NRAW
#define PK_NRAW 4  // measured on C5: 4/4 100.9 ms, 5/3 105.0, 5/4 104.9 per solve
#endif
#ifndef PK_NA
#define PK_NA 4
#endif
#ifndef PK_QB
#define PK_QB 4  // split-K partial slices a reduction thread keeps in flight (8: 86.5 ms per C5 solve against 79.2)
#endif
// one raw stage: A tile, B tile, and B's lo part right behind it, so that
// [B hi; B lo] is a single 128-row K-major operand: one N = 128 MMA
// computes A_hi·B_hi and A_hi·B_lo into the two adjacent accumulators
constexpr int RAW_FLOATS = (TM + 2 * RHS) * BK;
// + the epilogue's staging of the 64 x 128 Z / X values a tile updates
constexpr size_t PK_SMEM_BYTES = (size_t)PK_NRAW * RAW_FLOATS * 4 + (size_t)RHS * TM * 4 + 1024;
static_assert(PK_SMEM_BYTES <= 227 * 1024, "persistent ring exceeds shared memory");
static_assert(256 + 64 * PK_NA <= 512, "TMEM: two accumulators + the A ring");
constexpr int PK_TMEM_COLS = 512;
struct PkPipe {
  uint64_t full[PK_NRAW], rempty[PK_NRAW], conv[PK_NA], lempty[PK_NA];
  uint64_t tfull[2], tempty[2];
  uint32_t tmem;
};

__global__ void __launch_bounds__(NTW, 1)
    k_rebk_mrhs_persistent(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mAt,
                           const __grid_constant__ CUtensorMap mAtT,
                           const __grid_constant__ CUtensorMap mZt, const __grid_constant__ CUtensorMap mXt,
                           const __grid_constant__ CUtensorMap mUt, const __grid_constant__ CUtensorMap mRt,
                           const __grid_constant__ CUtensorMap mXst, const __grid_constant__ PkArgs a) {
  extern __shared__ float smem_raw[];
  float* smem = aligned_smem(smem_raw);
  __shared__ PkPipe P;
  __shared__ int s_crossed[RHS];
  __shared__ volatile int s_stop;
  __shared__ double s_wsum[4][RHS];  // stop check: per-warp column sums of (x - x*)^2 of a tile
  __shared__ float s_half[NRED];
  __shared__ float4 s_red4[NRED];
  __shared__ double s_errp[NRED / RHS][RHS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  if (warp == 0) umma::tmem_alloc<PK_TMEM_COLS>(&P.tmem);
  if (tid == 32) {
    for (int q = 0; q < PK_NRAW; ++q) {
      mbar_init(&P.full[q], 1);
      mbar_init(&P.rempty[q], 1);
    }
    for (int q = 0; q < PK_NA; ++q) {
      mbar_init(&P.conv[q], NCONV);
      mbar_init(&P.lempty[q], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&P.tfull[b], 1);
      mbar_init(&P.tempty[b], 4);
    }
    fence_mbar_init();
    s_stop = 0;
  }
  for (int c = tid; c < RHS; c += NTW) s_crossed[c] = (c < a.R) ? (a.iters[c] >= 0) : 1;
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = P.tmem;
  // end of global phase p = 4 (k - k_begin) + {0 A, 1 B, 2 C, 3 D}
  auto phase_end = [&](int64_t k, int ph) -> unsigned long long {
    return (unsigned long long)G * (unsigned long long)(4 * (k - a.k_begin) + ph + 1);
  };
  auto a_raw = [&](int q) { return smem + (size_t)q * RAW_FLOATS; };
  auto b_raw = [&](int q) { return smem + (size_t)q * RAW_FLOATS + TM * BK; };
  auto b_lo = [&](int q) { return smem + (size_t)q * RAW_FLOATS + (TM + RHS) * BK; };
  auto ta_hi = [&](int l) { return tmem + 256u + 64u * (uint32_t)l; };  // A hi; lo 32 columns on
  const int64_t k_last = a.k_end + 1;  // final round: P4(k_end) and its check only

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      uint32_t ph = 0;
      int it = 0, sc = 0;
      for (int64_t k = a.k_begin; k <= k_last; ++k) {
        for (int phase = 0; phase < 2; ++phase) {
          if (phase == 1) {
            if (k == k_last) break;
            gbar_wait(a.gbar, phase_end(k, 1));  // U ready (and the stop verdict)
            pk_stamp(a, k, 6);
            if (s_stop) break;
          } else if (k > a.k_begin) {
            gbar_wait(a.gbar, phase_end(k - 1, 3));  // R of the previous iteration ready
            pk_stamp(a, k, 7);
          }
          fence_proxy_async_global();
          PJob J;
          for (int j = 0; pk_job(a, phase, k, j, J); ++j) {
            const CUtensorMap* ma = (J.kind == 1 || J.kind == 4) ? &mAt : &mA;
            const CUtensorMap* mb = J.kind == 1 ? &mZt : (J.kind == 2 ? &mUt : (J.kind == 3 ? &mXt : &mRt));
            pk_jstamp(a, k, phase, j, 0);
            if (J.kind == 2 || J.kind == 4) {
              // the epilogue's read-modify-write rows (and x* on a check):
              // into L2 now, while this job's stages stream
              const CUtensorMap* my = J.kind == 2 ? &mZt : &mXt;
              for (int kk = 0; kk < TM / BK; ++kk) {
                tma_prefetch_l2_2d(my, J.row0 + kk * BK, 0);
                if (J.check) tma_prefetch_l2_2d(&mXst, J.row0 + kk * BK, 0);
              }
            }
            for (int kb = J.kb0; kb < J.kb1; ++kb, ++it) {
              const int q = it % PK_NRAW;
              if (it >= PK_NRAW) {
                mbar_wait(&P.rempty[q], (ph >> q) & 1u);
                ph ^= 1u << q;
              }
              pk_sstamp(a, k, sc, 0);
              mbar_arrive_expect_tx(&P.full[q], (TM + RHS) * BK * 4);
              const int kbe = kb;
              if (J.kind == 2)  // Z update: A_J through At, box 128 rows of z x 32 columns of J (L2-warm from P1)
                tma_load_2d(a_raw(q), &mAtT, J.row0, J.kc0 + kbe * BK, &P.full[q]);
              else
                tma_load_2d(a_raw(q), ma, J.kc0 + kbe * BK, J.row0, &P.full[q]);
              tma_load_2d(b_raw(q), mb, kbe * BK, 0, &P.full[q]);
              pk_sstamp(a, k, sc, 1);
              PK_SC_NEXT(k, sc);
            }
            pk_jstamp(a, k, phase, j, 1);
          }
          // A is immutable and the block sequence known: pull the next
          // phase's A boxes into L2 now, so HBM streams them during the
          // barriers and reductions in between (B operands are not final yet)
          if (a.prefetch) {
            const int nph = phase ^ 1;
            const int64_t nk = phase == 0 ? k : k + 1;
            if (nk <= k_last && !(nph == 1 && nk == k_last))
              for (int j = 0; pk_job(a, nph, nk, j, J); ++j) {
                const CUtensorMap* ma = (J.kind == 1 || J.kind == 4) ? &mAt : &mA;
                for (int kb = J.kb0; kb < J.kb1; ++kb) {
                  if (J.kind == 2) tma_prefetch_l2_2d(&mAtT, J.row0, J.kc0 + kb * BK);
                  else tma_prefetch_l2_2d(ma, J.kc0 + kb * BK, J.row0);
                }
              }
          }
        }
        if (s_stop) break;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      const uint32_t idesc = umma::idesc_tf32(TM, RHS);
      const uint32_t idesc2 = umma::idesc_tf32(TM, 2 * RHS);
      uint32_t phc = 0, pht = 0;
      int it = 0, jt = 0, sc = 0;
      for (int64_t k = a.k_begin; k <= k_last; ++k) {
        for (int phase = 0; phase < 2; ++phase) {
          if (phase == 1) {
            if (k == k_last) break;
            gbar_wait(a.gbar, phase_end(k, 1));
            if (s_stop) break;
          }
          PJob J;
          for (int j = 0; pk_job(a, phase, k, j, J); ++j, ++jt) {
            const int b = jt & 1;
            if (jt >= 2) {
              mbar_wait(&P.tempty[b], (pht >> b) & 1u);
              pht ^= 1u << b;
            }
            const uint32_t dh = tmem + b * 128, dl = dh + RHS;
            for (int kb = J.kb0; kb < J.kb1; ++kb, ++it) {
              const int q = it % PK_NRAW, l = it % PK_NA;
              mbar_wait(&P.conv[l], (phc >> l) & 1u);
              phc ^= 1u << l;
              pk_sstamp(a, k, sc, 5);
              if (kb == J.kb0) pk_jstamp(a, k, phase, j, 2);
              umma::fence_after_sync();
              const uint32_t tah = ta_hi(l), tal = tah + 32;
              for (int ks = 0; ks < BK / 8; ++ks) {
                // [B hi; B lo] as one N = 128 operand: D_hh | D_hl in one MMA
                const uint64_t bhl = umma::make_desc_sw128(smem_u32(b_raw(q)) + 32 * ks);
                const bool acc = kb > J.kb0 || ks > 0;
                if (!(a.dbg & 32)) {  // REBK_PK_DBG=32: no MMAs (timing experiments only)
                  umma::mma_tf32_ts(dh, tah + 8 * ks, bhl, idesc2, acc);
                  umma::mma_tf32_ts(dh, tal + 8 * ks, bhl, idesc, true);
                }
              }
              umma::commit(&P.rempty[q]);
              // with equally deep rings the raw stage and the TMEM-A slot of a
              // k-block are released by the same event: one commit serves both
              if (PK_NRAW != PK_NA) umma::commit(&P.lempty[l]);
              pk_sstamp(a, k, sc, 6);
              PK_SC_NEXT(k, sc);
            }
            umma::commit(&P.tfull[b]);
            pk_jstamp(a, k, phase, j, 3);
          }
        }
        if (s_stop) break;
      }
    }
  } else {
    // ---- converter warps (2-7) and epilogue warps (8-11); all of them run the reductions
    const bool conv = warp < EPI0;
    const int tr = tid - CONV0 * 32;  // 0 .. NRED-1
    uint32_t phf = 0, pht = 0, phl = 0;
    int it = 0, jt = 0, sc = 0;
    for (int64_t k = a.k_begin; k <= k_last; ++k) {
      for (int phase = 0; phase < 2; ++phase) {
        if (phase == 1 && k == k_last) break;
        PJob J;
        if (conv) {
          // warps 4-7: A rows of TMEM lane quadrant warp % 4 (hi = raw value,
          // the MMA truncates it to tf32; lo = exact remainder) -> TMEM;
          // warps 2-3: the B tile's lo part -> shared memory
          const bool aconv = warp >= 4;
          const int arow = 32 * (warp & 3) + lane;
          const int bt = tid - CONV0 * 32;  // 0..63 for the B warps
          for (int j = 0; pk_job(a, phase, k, j, J); ++j)
            for (int kb = J.kb0; kb < J.kb1; ++kb, ++it) {
              const int q = it % PK_NRAW, l = it % PK_NA;
              mbar_wait(&P.full[q], (phf >> q) & 1u);
              phf ^= 1u << q;
              if (tid == 128) pk_sstamp(a, k, sc, 2);
              if (a.dbg & 64) {  // REBK_PK_DBG=64: no conversion (timing experiments only)
                if (it >= PK_NA) {
                  mbar_wait(PK_NRAW != PK_NA ? &P.lempty[l] : &P.rempty[l], (phl >> l) & 1u);
                  phl ^= 1u << l;
                }
              } else if (aconv) {
                float hi[BK], lo[BK];
                if (J.kind == 2) {
                  // At box: row kk (column c_lo + kk of A) holds 128 z rows
                  const float* src = a_raw(q) + arow;
#pragma unroll
                  for (int kk = 0; kk < BK; ++kk) hi[kk] = src[kk * TM];
                } else {
                  const float* src = a_raw(q) + arow * BK;  // row r at r * 128 bytes, 16-byte chunks swizzled
#pragma unroll
                  for (int c = 0; c < BK / 4; ++c) {
                    const float4 v = *reinterpret_cast<const float4*>(src + (((c ^ arow) & 7) << 2));
                    hi[4 * c + 0] = v.x;
                    hi[4 * c + 1] = v.y;
                    hi[4 * c + 2] = v.z;
                    hi[4 * c + 3] = v.w;
                  }
                }
#pragma unroll
                for (int e = 0; e < BK; ++e) {
                  float h;
                  umma::split_tf32(hi[e], h, lo[e]);
                }
                if (it >= PK_NA) {  // the MMAs of stage it - PK_NA are done with slot l
                  mbar_wait(PK_NRAW != PK_NA ? &P.lempty[l] : &P.rempty[l], (phl >> l) & 1u);
                  phl ^= 1u << l;
                }
                const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
                umma::tmem_st32(ta_hi(l) + lane_base, hi);
                umma::tmem_st32(ta_hi(l) + 32 + lane_base, lo);
                umma::tmem_wait_st();
                umma::fence_before_sync();
              } else {
                constexpr int B4 = RHS * BK / 4, PERB = B4 / 64;
                static_assert(B4 % 64 == 0, "B converter split");
                const float4* srcB = reinterpret_cast<const float4*>(b_raw(q));
                float4 v[PERB];
#pragma unroll
                for (int i = 0; i < PERB; ++i) v[i] = srcB[bt + i * 64];
                float4* dstB = reinterpret_cast<float4*>(b_lo(q));
#pragma unroll
                for (int i = 0; i < PERB; ++i) {
                  float4 lo;
                  float h;
                  umma::split_tf32(v[i].x, h, lo.x);
                  umma::split_tf32(v[i].y, h, lo.y);
                  umma::split_tf32(v[i].z, h, lo.z);
                  umma::split_tf32(v[i].w, h, lo.w);
                  dstB[bt + i * 64] = lo;
                }
                fence_proxy_async();
              }
              __syncwarp();
              if (tid == 128) pk_sstamp(a, k, sc, 3);
              if (tid == 64) pk_sstamp(a, k, sc, 4);
              if (lane == 0 && warp >= 5) pk_sstamp(a, k, sc, 3 + warp);  // 8, 9, 10: A converter warps 5, 6, 7
              if (tid == 96) pk_sstamp(a, k, sc, 11);                     // the second B converter warp
              PK_SC_NEXT(k, sc);
              if (lane == 0) mbar_arrive(&P.conv[l]);
            }
        } else {
          const int ew = warp & 3, rlane = ew * 32;
          for (int j = 0; pk_job(a, phase, k, j, J); ++j, ++jt) {
            const int b = jt & 1;
            const int row = rlane + lane;
            const bool any = J.kb1 > J.kb0;
            const bool mode0 = J.kind == 1 || J.kind == 3;
            float* part = J.kind == 1 ? a.part1 : a.part3;
            float* Y = J.kind == 2 ? a.Zt : a.Xt;
            const int64_t ldy = J.kind == 2 ? a.m : a.n;
            const int r = J.row0 + row;
            const bool live = !mode0 && r < ldy;
            const bool chk = J.check && live && !(a.dbg & 16);
            // all 64 values of the row this thread updates (final for this
            // phase) are copied to shared memory while the MMAs run (cp.async:
            // no registers held, one round trip); x* chunks come through
            // registers, chunk c+1 while chunk c is applied
            float* s_y = smem + (size_t)PK_NRAW * RAW_FLOATS;  // [RHS][TM], this thread's row only
            float xcur[16], xnext[16];
            if (live) {
#pragma unroll 8
              for (int q = 0; q < RHS; ++q)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s_y + q * TM + row)),
                             "l"(Y + (size_t)q * ldy + r)
                             : "memory");
              asm volatile("cp.async.commit_group;" ::: "memory");
            }
            if (chk) {
#pragma unroll
              for (int q = 0; q < 16; ++q) xcur[q] = __ldg(a.Xst + (size_t)q * ldy + r);
            }
            mbar_wait(&P.tfull[b], (pht >> b) & 1u);
            pht ^= 1u << b;
            if (tid == EPI0 * 32) pk_jstamp(a, k, phase, j, 4);
            umma::fence_after_sync();
            if (live) asm volatile("cp.async.wait_all;" ::: "memory");
            const uint32_t base = tmem + ((uint32_t)rlane << 16) + b * 128;
#pragma unroll
            for (int c0 = 0; c0 < RHS; c0 += 16) {
              float ycur[16];
              if (c0 + 16 < RHS) {
                if (chk) {
#pragma unroll
                  for (int q = 0; q < 16; ++q) xnext[q] = __ldg(a.Xst + (size_t)(c0 + 16 + q) * ldy + r);
                }
              }
              float h[16], l[16];
              {
                uint32_t rh[16], rl[16];
                umma::tmem_ld16_nowait(base + c0, rh);
                umma::tmem_ld16_nowait(base + RHS + c0, rl);
                umma::tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                  h[q] = __uint_as_float(rh[q]);
                  l[q] = __uint_as_float(rl[q]);
                }
              }
              if (mode0) {
                // partial slices are stored [slice][c][256 rows]: for a fixed
                // right-hand side the warp's 32 rows are one 128-byte line
                // (row-major [row][c] was 32 partial sectors per store)
                float* dst = part + ((size_t)J.slot * RHS + c0) * 256 + J.prow + row;
#pragma unroll
                for (int q = 0; q < 16; ++q) __stcg(dst + (size_t)q * 256, any ? h[q] + l[q] : 0.f);
              } else {
                if (live && any) {
#pragma unroll
                  for (int q = 0; q < 16; ++q) {
                    ycur[q] = s_y[(c0 + q) * TM + row] - J.s * (h[q] + l[q]);
                    __stcg(Y + (size_t)(c0 + q) * ldy + r, ycur[q]);
                  }
                } else {
#pragma unroll
                  for (int q = 0; q < 16; ++q) ycur[q] = live ? s_y[(c0 + q) * TM + row] : 0.f;
                }
                if (J.check) {
                  // Σ over the warp's 32 rows of (x - x*)^2, 8 columns at a
                  // time by a transposing butterfly (fixed order; after the
                  // xor 16/8/4 halvings lane L holds column (L>>4&1)*4 +
                  // (L>>3&1)*2 + (L>>2&1), then xor 2 and 1 finish the sum);
                  // the four warp sums are added in order after the tile
#pragma unroll
                  for (int hh = 0; hh < 2; ++hh) {
                    double v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                      const double d = chk ? (double)ycur[8 * hh + q] - (double)xcur[8 * hh + q] : 0.0;
                      v[q] = d * d;
                    }
#pragma unroll
                    for (int m = 16, n = 8; m >= 4; m >>= 1, n >>= 1) {
                      const bool up = (lane & m) != 0;
#pragma unroll
                      for (int i = 0; i < n / 2; ++i) {
                        const double send = up ? v[i] : v[i + n / 2];
                        const double keep = up ? v[i + n / 2] : v[i];
                        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                      }
                    }
                    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
                    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
                    if ((lane & 3) == 0) {
                      const int col = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                      s_wsum[ew][c0 + 8 * hh + col] = v[0];
                    }
                  }
                }
              }
#pragma unroll
              for (int q = 0; q < 16; ++q) xcur[q] = xnext[q];
            }
            fence_proxy_async_global();
            umma::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(&P.tempty[b]);
            if (tid == EPI0 * 32) pk_jstamp(a, k, phase, j, 5);
            if (J.check) {
              named_bar(1, 128);
              const int c = tr - (EPI0 - CONV0) * 32;
              if (c < RHS) a.errpart[(size_t)J.slot * RHS + c] = ((s_wsum[0][c] + s_wsum[1][c]) + s_wsum[2][c]) + s_wsum[3][c];
            }
          }
          // this CTA's part of the phase is written: arrive
          named_bar(1, 128);
          if (tid == EPI0 * 32) {
            pk_stamp(a, k, phase == 0 ? 0 : 3);
            // the counter is shared by all phases: a CTA with no jobs in this
            // phase must not arrive before the previous phase has ended
            // everywhere, or its arrival would stand in for a late one there
            if (phase == 1) gbar_wait(a.gbar, phase_end(k, 1));
            else if (k > a.k_begin) gbar_wait(a.gbar, phase_end(k - 1, 3));
            gbar_arrive(a.gbar);
            pk_stamp(a, k, phase == 0 ? 8 : 10);
          }
        }
        // ---- reduction phase (B after A, D after C): one thread polls
#ifdef PK_ALLPOLL
        gbar_wait(a.gbar, phase_end(k, phase == 0 ? 0 : 2));
#else
        if (tr == 0) {
          gbar_wait(a.gbar, phase_end(k, phase == 0 ? 0 : 2));
          pk_stamp(a, k, phase == 0 ? 1 : 4);
        }
#endif
        __syncwarp();
        named_bar(2, NRED);
        if (tr == 0) pk_stamp(a, k, phase == 0 ? 9 : 11);
        const int b = blockIdx.x;
        if (phase == 0) {
          // stop check of iteration k-1 (every CTA, same bits)
          if (k - 1 >= a.k_begin && pk_is_check(a, k - 1)) {
            // per-column Σ over the nt4 tile partials: NRED / RHS threads per
            // column take tiles pp, pp + NP, ... (loads issued together), then a
            // fixed-order combine, so the check costs one L2 round trip
            {
              constexpr int NP = NRED / RHS;
              const int c = tr % RHS, pp = tr / RHS;
              if (pp < NP) {
                double s = 0.0;
                if (c < a.R) {
                  for (int t0 = pp; t0 < a.nt4; t0 += 8 * NP) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                      v[u] = (t0 + u * NP < a.nt4) ? ld_cg_f64(a.errpart + (size_t)(t0 + u * NP) * RHS + c) : 0.0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) s += v[u];
                  }
                }
                s_errp[pp][c] = s;
              }
            }
            named_bar(2, NRED);
            if (tr < a.R) {
              double s = 0.0;
#pragma unroll
              for (int pp = 0; pp < NRED / RHS; ++pp) s += s_errp[pp][tr];
              const double e = sqrt(s);
              if (!s_crossed[tr] && e <= a.tol[tr]) {
                s_crossed[tr] = 1;
                if (b == 0) {
                  a.iters[tr] = k - 1;
                  a.errs_at[tr] = e;
                }
              }
            }
            named_bar(2, NRED);
            if (tr == 0) {
              int all = 1;
              for (int c = 0; c < a.R; ++c) all &= s_crossed[c];
              if (all) {
                s_stop = 1;
                if (b == 0) {
                  *a.k_final = k - 1;
                  *a.stopped = 1;
                }
              }
            }
          }
          // U = Σ_q part1[q] (slices stored [q][c][256]): 128 chunks of 128
          // entries (half a right-hand side's row of Ut); the chunk's 32 float4
          // groups get NRED / 32 threads each, thread `sub` summing slices
          // [ns1*sub/T, ns1*(sub+1)/T) with all its loads in flight, then the T
          // range sums are added in order
          if (a.extended && k <= a.k_end) {
            const Plan& pl = a.plan[k - a.k_begin];
            const int nJ = pl.c_hi - pl.c_lo;
            constexpr int T = NRED / 32;
            const int gi = tr / T, sub = tr % T;
            for (int ch = b; ch < 256 * RHS / 128; ch += G) {
              const int c = ch >> 1, j4 = (ch & 1) * 128 + gi * 4;
              float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
              if (j4 < nJ) {
                const int q0 = (a.ns1 * sub) / T, q1 = (a.ns1 * (sub + 1)) / T;
                const float4* src = reinterpret_cast<const float4*>(a.part1 + (size_t)c * 256 + j4);
                constexpr int QB = PK_QB;
                for (int qb = q0; qb < q1; qb += QB) {
                  float4 v[QB];
#pragma unroll
                  for (int u = 0; u < QB; ++u)
                    if (qb + u < q1)
                      asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                                   : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                                   : "l"(src + (size_t)(qb + u) * (256 * RHS / 4))
                                   : "memory");
#pragma unroll
                  for (int u = 0; u < QB; ++u)
                    if (qb + u < q1) {
                      acc.x += v[u].x;
                      acc.y += v[u].y;
                      acc.z += v[u].z;
                      acc.w += v[u].w;
                    }
                }
              }
              s_red4[tr] = acc;
              named_bar(2, NRED);
              if (sub == 0) {
                for (int t = 1; t < T; ++t) {
                  const float4 w = s_red4[tr + t];
                  acc.x += w.x;
                  acc.y += w.y;
                  acc.z += w.z;
                  acc.w += w.w;
                }
                // rows past |J| are K padding of the z update: zero
                float4 o;
                o.x = j4 + 0 < nJ ? acc.x : 0.f;
                o.y = j4 + 1 < nJ ? acc.y : 0.f;
                o.z = j4 + 2 < nJ ? acc.z : 0.f;
                o.w = j4 + 3 < nJ ? acc.w : 0.f;
                *reinterpret_cast<float4*>(a.Ut + (size_t)c * 256 + j4) = o;
              }
              named_bar(2, NRED);
            }
          }
        } else {
          // R = ((Σ_q part3[q]) - B_I) + Z_I  (solvers.py:291-293 order), zero past |I|;
          // float4 groups along the rows as for U, b_I and z_I fetched before the partials
          const Plan& pl = a.plan[k - a.k_begin];
          const int nI = pl.r_hi - pl.r_lo;
          constexpr int T = NRED / 32;
          const int gi = tr / T, sub = tr % T;
          for (int ch = b; ch < 256 * RHS / 128; ch += G) {
            const int c = ch >> 1, i4 = (ch & 1) * 128 + gi * 4;
            const bool valid = i4 < nI;
            float bt[4] = {0.f, 0.f, 0.f, 0.f}, zt[4] = {0.f, 0.f, 0.f, 0.f};
            if (sub == 0 && valid) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (i4 + u < nI) {
                  bt[u] = ld_cg_f32(a.Bt + (size_t)c * a.m + pl.r_lo + i4 + u);
                  if (a.extended) zt[u] = ld_cg_f32(a.Zt + (size_t)c * a.m + pl.r_lo + i4 + u);
                }
            }
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            if (valid) {
              const int q0 = (a.ns3 * sub) / T, q1 = (a.ns3 * (sub + 1)) / T;
              const float4* src = reinterpret_cast<const float4*>(a.part3 + (size_t)c * 256 + i4);
              constexpr int QB = PK_QB;
              for (int qb = q0; qb < q1; qb += QB) {
                float4 v[QB];
#pragma unroll
                for (int u = 0; u < QB; ++u)
                  if (qb + u < q1)
                    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                                 : "l"(src + (size_t)(qb + u) * (256 * RHS / 4))
                                 : "memory");
#pragma unroll
                for (int u = 0; u < QB; ++u)
                  if (qb + u < q1) {
                    acc.x += v[u].x;
                    acc.y += v[u].y;
                    acc.z += v[u].z;
                    acc.w += v[u].w;
                  }
              }
            }
            s_red4[tr] = acc;
            named_bar(2, NRED);
            if (sub == 0) {
              for (int t = 1; t < T; ++t) {
                const float4 w = s_red4[tr + t];
                acc.x += w.x;
                acc.y += w.y;
                acc.z += w.z;
                acc.w += w.w;
              }
              const float sum[4] = {acc.x, acc.y, acc.z, acc.w};
              float o[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                float v = 0.f;
                if (i4 + u < nI) {
                  v = sum[u] - bt[u];
                  if (a.extended) v += zt[u];
                }
                o[u] = v;
              }
              *reinterpret_cast<float4*>(a.Rt + (size_t)c * 256 + i4) = make_float4(o[0], o[1], o[2], o[3]);
            }
            named_bar(2, NRED);
          }
        }
        fence_proxy_async_global();
        named_bar(2, NRED);
        if (tr == 0) {
          pk_stamp(a, k, phase == 0 ? 2 : 5);
          gbar_arrive(a.gbar);
        }
        if (phase == 0 && (s_stop || k == k_last)) break;
      }
      if (s_stop || k == k_last) break;
    }
    if (tr == 0 && blockIdx.x == 0 && !s_stop) *a.k_final = a.k_end;
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<PK_TMEM_COLS>(tmem);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  }
  return fn;
}
// K-major operand view of a row-major fp32 matrix (rows x kdim, leading dim
// ld): box of 32 along K x box_rows with the 128-byte swizzle
static bool encode_kmajor(CUtensorMap* map, const float* base, int64_t rows, int64_t kdim, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encoder();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// At (n x m, leading dim ld) read as the Z update's A operand: box of 128
// consecutive z rows (At's inner dimension) x 32 columns of the block, no
// swizzle (512-byte rows); the converter warps transpose it into TMEM
static bool encode_at_rows(CUtensorMap* map, const float* At, int64_t n, int64_t m, int64_t ld) {
  EncodeTiledFn fn = encoder();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)TM, (cuuint32_t)BK};
  cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)At, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tc

cudaError_t mrhs_transpose_a(const float* A, int64_t m, int64_t n, int64_t lda, float* At, int64_t ldat,
                             cudaStream_t st) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32)), block(32, 8);
  tc::k_transpose<<<grid, block, 0, st>>>(A, m, n, lda, At, ldat);
  return cudaGetLastError();
}

bool mrhs_tc_supported(int64_t m, int64_t n, int R, int nJmax, int nImax) {
  return R >= 1 && R <= tc::RHS && m % 4 == 0 && n % 4 == 0 && nJmax <= 256 && nImax <= 256 && tc::encoder() != nullptr;
}

#define TC_TRY(expr)                                                     \
  do {                                                                   \
    cudaError_t _e = (expr);                                             \
    if (_e != cudaSuccess) {                                             \
      snprintf(errbuf, errlen, "%s: %s", #expr, cudaGetErrorString(_e)); \
      return -2;                                                         \
    }                                                                    \
  } while (0)

// Same contract as run_mrhs (rebk_mrhs.cu): per-column stopping on the
// device, chunks of 64 iterations captured as CUDA graphs, exact stop state
// by checkpoint + replay.  w.B/X/Z/Xs are row-major (rows x 64) on entry and
// exit; inside they are kept transposed.
int run_mrhs_tc(const MrhsRun& w, const SampleParams& sp_template, int64_t* iters_out, double* errs_out,
                double* loop_ms, int64_t* k_final, char* errbuf, size_t errlen, cudaStream_t stream) {
  using namespace tc;
  const rebk_cfg* cfg = w.cfg;
  const int R = w.R;
  const int64_t m = w.m, n = w.n;
  const bool checking = cfg->stop_mode == 0;
  int nJmax = 1, nImax = 1;
  for (int64_t b = 0; b < cfg->n_row_blocks; ++b) nImax = std::max<int>(nImax, (int)(cfg->row_ptr[b + 1] - cfg->row_ptr[b]));
  if (w.extended)
    for (int64_t b = 0; b < cfg->n_col_blocks; ++b)
      nJmax = std::max<int>(nJmax, (int)(cfg->col_ptr[b + 1] - cfg->col_ptr[b]));
  for (int64_t b = 0; b < cfg->n_row_blocks; ++b)
    if (cfg->row_ptr[b] % 4) {
      snprintf(errbuf, errlen, "tensor-core multi-RHS path needs row blocks starting at multiples of 4");
      return -3;
    }
  if (w.extended)
    for (int64_t b = 0; b < cfg->n_col_blocks; ++b)
      if (cfg->col_ptr[b] % 4) {
        snprintf(errbuf, errlen, "tensor-core multi-RHS path needs column blocks starting at multiples of 4");
        return -3;
      }
  const int ldu = 256, ldr = 256;  // Ut / Rt padded to whole K-blocks (zeros)
  float *Zt = nullptr, *Xt, *Bt, *Xst = nullptr, *Ut, *Rt, *part, *Xsnap, *Zsnap = nullptr;
  double *d_tol, *d_errs_at, *d_cpart;
  int64_t* d_iters;
  int32_t* d_ndone;
  Plan* d_plan;
  const int G1 = 148, G3 = 40;  // CTAs (K slices) of the two split-K products; each does every row tile
  const int nchk = (int)((n + kChk - 1) / kChk);
  // the transposed arrays always have 64 rows (the MMA N); rows R..63 are zero
  TC_TRY(cudaMallocAsync((void**)&Xt, sizeof(float) * RHS * n, stream));
  TC_TRY(cudaMallocAsync((void**)&Bt, sizeof(float) * RHS * m, stream));
  if (w.extended) TC_TRY(cudaMallocAsync((void**)&Zt, sizeof(float) * RHS * m, stream));
  if (w.Xs) TC_TRY(cudaMallocAsync((void**)&Xst, sizeof(float) * RHS * n, stream));
  TC_TRY(cudaMallocAsync((void**)&Ut, sizeof(float) * RHS * ldu, stream));
  TC_TRY(cudaMallocAsync((void**)&Rt, sizeof(float) * RHS * ldr, stream));
  TC_TRY(cudaMallocAsync((void**)&part, sizeof(float) * (size_t)std::max(G1, G3) * 256 * RHS, stream));
  TC_TRY(cudaMemsetAsync(part, 0, sizeof(float) * (size_t)std::max(G1, G3) * 256 * RHS, stream));
  TC_TRY(cudaMallocAsync((void**)&Xsnap, sizeof(float) * RHS * n, stream));
  if (w.extended) TC_TRY(cudaMallocAsync((void**)&Zsnap, sizeof(float) * RHS * m, stream));
  TC_TRY(cudaMallocAsync((void**)&d_tol, sizeof(double) * R, stream));
  TC_TRY(cudaMallocAsync((void**)&d_errs_at, sizeof(double) * R, stream));
  TC_TRY(cudaMallocAsync((void**)&d_cpart, sizeof(double) * R * nchk, stream));
  TC_TRY(cudaMallocAsync((void**)&d_iters, sizeof(int64_t) * R, stream));
  TC_TRY(cudaMallocAsync((void**)&d_ndone, sizeof(int32_t), stream));
  const int64_t CH = 64;
  TC_TRY(cudaMallocAsync((void**)&d_plan, sizeof(Plan) * CH, stream));
  dim3 tb(32, 8);
  k_to_t<<<dim3((unsigned)((n + 31) / 32), RHS / 32), tb, 0, stream>>>(w.X, n, R, Xt, n);
  k_to_t<<<dim3((unsigned)((m + 31) / 32), RHS / 32), tb, 0, stream>>>(w.B, m, R, Bt, m);
  if (w.extended) k_to_t<<<dim3((unsigned)((m + 31) / 32), RHS / 32), tb, 0, stream>>>(w.Z, m, R, Zt, m);
  if (Xst) k_to_t<<<dim3((unsigned)((n + 31) / 32), RHS / 32), tb, 0, stream>>>(w.Xs, n, R, Xst, n);
  TC_TRY(cudaGetLastError());
  std::vector<double> tol(R);
  for (int c = 0; c < R; ++c) tol[c] = w.tols ? w.tols[c] : cfg->tol;
  TC_TRY(cudaMemcpyAsync(d_tol, tol.data(), sizeof(double) * R, cudaMemcpyHostToDevice, stream));
  TC_TRY(cudaMemsetAsync(d_iters, 0xff, sizeof(int64_t) * R, stream));
  TC_TRY(cudaMemsetAsync(d_ndone, 0, sizeof(int32_t), stream));
  TC_TRY(cudaMemsetAsync(d_errs_at, 0, sizeof(double) * R, stream));

  // tensor maps: A and At views (128-row boxes), iterate views (64-row boxes)
  CUtensorMap mA, mAt, mAtT, mZt, mXt, mUt, mRt;
  bool ok = encode_kmajor(&mA, w.A, m, n, w.lda, TM) && encode_kmajor(&mXt, Xt, RHS, n, n, RHS) &&
            encode_kmajor(&mUt, Ut, RHS, ldu, ldu, RHS) && encode_kmajor(&mRt, Rt, RHS, ldr, ldr, RHS);
  if (w.extended) ok = ok && encode_kmajor(&mAt, w.At, n, m, w.ldat, TM) && encode_kmajor(&mZt, Zt, RHS, m, m, RHS);
  else ok = ok && encode_kmajor(&mAt, w.At, n, m, w.ldat, TM);
  ok = ok && encode_at_rows(&mAtT, w.At, n, m, w.ldat);
  CUtensorMap mXst = mXt;
  if (ok && Xst) ok = encode_kmajor(&mXst, Xst, RHS, n, n, RHS);
  if (!ok) {
    snprintf(errbuf, errlen, "tensor map encoding failed");
    return -2;
  }
  TC_TRY(cudaFuncSetAttribute(k_gemm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
  TC_TRY(cudaFuncSetAttribute(k_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);

  auto launch_check = [&](int64_t k) -> cudaError_t {
    k_check_part<<<dim3(nchk, R), 256, 0, stream>>>(Xt, Xst, n, d_cpart);
    k_check_final<<<(R + 63) / 64, 64, 0, stream>>>(d_cpart, nchk, R, d_tol, k, d_iters, d_errs_at, d_ndone);
    return cudaGetLastError();
  };
  const int nkb_m = (int)((m + BK - 1) / BK), nkb_n = (int)((n + BK - 1) / BK);
  const char* dbg_env = getenv("REBK_TC_DBG");  // experiments: 1 skip lo split, 2 skip MMAs, 4 L2 prefetch
  const int dbg = dbg_env ? atoi(dbg_env) : 0;
  if (TM * 2 > 256 || RHS % 32) return -3;
  auto enqueue_iter = [&](const Plan& pl, int64_t k, bool do_check) -> cudaError_t {
    const int nJ = pl.c_hi - pl.c_lo, nI = pl.r_hi - pl.r_lo;
    if (w.extended) {
      const int ns = G1;
      k_gemm<0><<<ns, NTW, SMEM_BYTES, stream>>>(mAt, mZt, 0, pl.c_lo, nJ, nkb_m, ns, 0.f, part, 0, dbg);
      k_reduce_u<<<dim3(ldu, RHS / 32), 256, 0, stream>>>(part, ns, nJ, ldu, Ut);
      k_gemm<1><<<std::min(nsm, (int)((m + TM - 1) / TM)), NTW, SMEM_BYTES, stream>>>(
          mA, mUt, pl.c_lo, 0, (int)m, (nJ + BK - 1) / BK, 0, (float)pl.c_scale, Zt, m, dbg);
    }
    const int ns3 = G3;
    k_gemm<0><<<ns3, NTW, SMEM_BYTES, stream>>>(mA, mXt, 0, pl.r_lo, nI, nkb_n, ns3, 0.f, part, 0, dbg);
    k_reduce_r<<<dim3(ldr, RHS / 32), 256, 0, stream>>>(part, ns3, nI, ldr, Bt, Zt, m, pl.r_lo, Rt);
    k_gemm<1><<<std::min(nsm, (int)((n + TM - 1) / TM)), NTW, SMEM_BYTES, stream>>>(
        mAt, mRt, pl.r_lo, 0, (int)n, (nI + BK - 1) / BK, 0, (float)pl.r_scale, Xt, n, dbg);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && do_check) e = launch_check(k);
    return e;
  };

  // persistent whole-run kernel (default): one cooperative launch per chunk
  // of up to 2^20 iterations; REBK_MRHS_PK=0 selects the per-product kernels
  const char* pk_env = getenv("REBK_MRHS_PK");
  const int G = nsm & ~1;
  const int nt2 = (int)((m + TM - 1) / TM), nt4 = (int)((n + TM - 1) / TM);
  bool use_pk = !(pk_env && pk_env[0] == '0') && G >= 2 && nt4 <= G && !(dbg & 3);
  if (use_pk) {
    TC_TRY(cudaFuncSetAttribute(k_rebk_mrhs_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PK_SMEM_BYTES));
    int occ = 0;
    TC_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rebk_mrhs_persistent, NTW, PK_SMEM_BYTES));
    use_pk = occ >= 1;
  }

  cudaEvent_t ev0, ev1;
  TC_TRY(cudaEventCreate(&ev0));
  TC_TRY(cudaEventCreate(&ev1));
  TC_TRY(cudaEventRecord(ev0, stream));
  int64_t K = cfg->max_iters;
  bool all_done = false;
  if (checking) {
    TC_TRY(launch_check(0));
    int32_t nd = 0;
    TC_TRY(cudaMemcpyAsync(&nd, d_ndone, sizeof nd, cudaMemcpyDeviceToHost, stream));
    TC_TRY(cudaStreamSynchronize(stream));
    if (nd == R) {
      all_done = true;
      K = 0;
    }
  }
  if (use_pk && !all_done && cfg->max_iters > 0) {
    PkArgs pa{};
    pa.m = (int)m;
    pa.n = (int)n;
    pa.nkb_m = nkb_m;
    pa.nkb_n = nkb_n;
    pa.extended = w.extended;
    pa.checking = checking;
    pa.stride = (int)cfg->check_stride;
    pa.max_iters = cfg->max_iters;
    pa.ns1 = std::max(1, std::min(G / 2, nkb_m));
    pa.p3_first = 0;
    if (w.extended && nt2 % G != 0) pa.p3_first = std::min(G - 2, ((nt2 % G) + 1) & ~1);
    pa.ns3 = std::max(1, std::min((G - pa.p3_first) / 2, nkb_n));
    pa.nt2 = nt2;
    pa.nt4 = nt4;
    pa.R = R;
    pa.Zt = Zt;
    pa.Xt = Xt;
    pa.Ut = Ut;
    pa.Rt = Rt;
    pa.Bt = Bt;
    pa.Xst = Xst;
    pa.tol = d_tol;
    pa.iters = d_iters;
    pa.errs_at = d_errs_at;
    float *p1 = nullptr, *p3 = nullptr;
    double* ep = nullptr;
    int64_t* d_kf = nullptr;
    int32_t* d_stopped = nullptr;
    unsigned long long* d_gbar = nullptr;
    Plan* d_plan_all = nullptr;
    const int64_t CHK = std::min<int64_t>(cfg->max_iters, (int64_t)1 << 20);
    TC_TRY(cudaMallocAsync((void**)&p1, sizeof(float) * (size_t)pa.ns1 * 256 * RHS, stream));
    TC_TRY(cudaMallocAsync((void**)&p3, sizeof(float) * (size_t)pa.ns3 * 256 * RHS, stream));
    TC_TRY(cudaMallocAsync((void**)&ep, sizeof(double) * (size_t)nt4 * RHS, stream));
    TC_TRY(cudaMallocAsync((void**)&d_kf, sizeof(int64_t), stream));
    TC_TRY(cudaMallocAsync((void**)&d_stopped, sizeof(int32_t), stream));
    TC_TRY(cudaMallocAsync((void**)&d_gbar, sizeof(unsigned long long), stream));
    TC_TRY(cudaMallocAsync((void**)&d_plan_all, sizeof(Plan) * CHK, stream));
    TC_TRY(cudaMemsetAsync(d_stopped, 0, sizeof(int32_t), stream));
    pa.part1 = p1;
    pa.part3 = p3;
    pa.errpart = ep;
    pa.k_final = d_kf;
    pa.stopped = d_stopped;
    pa.gbar = d_gbar;
    pa.plan = d_plan_all;
    const char* pf_env = getenv("REBK_PK_PREFETCH");
    pa.prefetch = pf_env ? atoi(pf_env) : 1;
    const char* pdbg = getenv("REBK_PK_DBG");
    pa.dbg = pdbg ? atoi(pdbg) : 0;
    const char* tr_env = getenv("REBK_PK_TRACE");
    pa.trace_n = tr_env ? atoi(tr_env) : 0;
    pa.trace_k0 = 100;
    unsigned long long* d_tr = nullptr;
    if (pa.trace_n > 0) {
      TC_TRY(cudaMallocAsync((void**)&d_tr, sizeof(unsigned long long) * pa.trace_n * G * PK_TRACE_SLOTS, stream));
      TC_TRY(cudaMemsetAsync(d_tr, 0, sizeof(unsigned long long) * pa.trace_n * G * PK_TRACE_SLOTS, stream));
      pa.trace = d_tr;
      TC_TRY(cudaMallocAsync((void**)&pa.trace2, sizeof(unsigned long long) * 2 * 2 * 4 * 8, stream));
      TC_TRY(cudaMemsetAsync(pa.trace2, 0, sizeof(unsigned long long) * 2 * 2 * 4 * 8, stream));
#ifdef PK_STAGE_TRACE
      TC_TRY(cudaMallocAsync((void**)&pa.trace3, sizeof(long long) * PK_STAGE_TRACE_N * 12, stream));
      TC_TRY(cudaMemsetAsync(pa.trace3, 0, sizeof(long long) * PK_STAGE_TRACE_N * 12, stream));
#endif
    }
    for (int64_t k0 = 1; k0 <= cfg->max_iters; k0 += CHK) {
      const int64_t cnt = std::min(CHK, cfg->max_iters - k0 + 1);
      TC_TRY(launch_sample_plan(sp_template, k0, cnt, d_plan_all, nullptr, stream));
      TC_TRY(cudaMemsetAsync(d_gbar, 0, sizeof(unsigned long long), stream));
      pa.k_begin = k0;
      pa.k_end = k0 + cnt - 1;
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(G);
      lc.blockDim = dim3(NTW);
      lc.dynamicSmemBytes = PK_SMEM_BYTES;
      lc.stream = stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      TC_TRY(cudaLaunchKernelEx(&lc, k_rebk_mrhs_persistent, mA, mAt, mAtT, w.extended ? mZt : mXt, mXt,
                                mUt, mRt, mXst, pa));
      int32_t st = 0;
      int64_t kf = 0;
      TC_TRY(cudaMemcpyAsync(&st, d_stopped, sizeof st, cudaMemcpyDeviceToHost, stream));
      TC_TRY(cudaMemcpyAsync(&kf, d_kf, sizeof kf, cudaMemcpyDeviceToHost, stream));
      TC_TRY(cudaStreamSynchronize(stream));
      K = kf;
      if (st) break;
    }
    if (d_tr) {
      std::vector<unsigned long long> h((size_t)pa.trace_n * G * PK_TRACE_SLOTS);
      TC_TRY(cudaMemcpy(h.data(), d_tr, h.size() * 8, cudaMemcpyDeviceToHost));
      const char* fn = getenv("REBK_PK_TRACE_FILE");
      FILE* f = fopen(fn ? fn : "pk_trace.bin", "wb");
      if (f) {
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
      }
      cudaFree(d_tr);
      std::vector<unsigned long long> h2(2 * 2 * 4 * 8);
      TC_TRY(cudaMemcpy(h2.data(), pa.trace2, h2.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long t0 = 0;
      for (auto v : h2)
        if (v && (!t0 || v < t0)) t0 = v;
      for (int sel = 0; sel < 2; ++sel)
        for (int ph = 0; ph < 2; ++ph)
          for (int jj = 0; jj < 4; ++jj) {
            const unsigned long long* e = &h2[((sel * 2 + ph) * 4 + jj) * 8];
            if (!e[0]) continue;
            fprintf(stderr, "[pk job] cta %d phase %c job %d:", sel ? 120 : 0, ph ? 'C' : 'A', jj);
            for (int ev = 0; ev < 6; ++ev) fprintf(stderr, " %8.2f", e[ev] ? (e[ev] - t0) * 1e-3 : -1.0);
            fprintf(stderr, "\n");
          }
      cudaFree(pa.trace2);
#ifdef PK_STAGE_TRACE
      std::vector<long long> h3(PK_STAGE_TRACE_N * 12);
      TC_TRY(cudaMemcpy(h3.data(), pa.trace3, h3.size() * 8, cudaMemcpyDeviceToHost));
      long long c0 = 0;
      for (int i = 0; i < PK_STAGE_TRACE_N; ++i)
        if (h3[i * 12 + 1] && (!c0 || h3[i * 12 + 1] < c0)) c0 = h3[i * 12 + 1];
      fprintf(stderr, "[pk stage] cycles since the first issue: free issued | A full, A stored (warp 4) | B done (warp 2) | MMA conv, committed | - | A stored warps 5 6 7 | B done warp 3\n");
      for (int i = 0; i < PK_STAGE_TRACE_N; ++i) {
        if (!h3[i * 12 + 1]) continue;
        fprintf(stderr, "[pk stage] %3d:", i);
        for (int ev = 0; ev < 12; ++ev) fprintf(stderr, " %7lld", h3[i * 12 + ev] ? h3[i * 12 + ev] - c0 : -1LL);
        fprintf(stderr, "\n");
      }
      cudaFree(pa.trace3);
#endif
    }
    all_done = true;  // skip the per-product loop below
    for (void* ptr : {(void*)p1, (void*)p3, (void*)ep, (void*)d_kf, (void*)d_stopped, (void*)d_gbar, (void*)d_plan_all})
      cudaFreeAsync(ptr, stream);
  }
  std::vector<Plan> hplan(CH);
  for (int64_t k0 = 1; !all_done && k0 <= cfg->max_iters; k0 += CH) {
    const int64_t cnt = std::min(CH, cfg->max_iters - k0 + 1);
    TC_TRY(launch_sample_plan(sp_template, k0, cnt, d_plan, nullptr, stream));
    TC_TRY(cudaMemcpyAsync(hplan.data(), d_plan, sizeof(Plan) * cnt, cudaMemcpyDeviceToHost, stream));
    TC_TRY(cudaStreamSynchronize(stream));
    if (checking) {
      TC_TRY(cudaMemcpyAsync(Xsnap, Xt, sizeof(float) * n * RHS, cudaMemcpyDeviceToDevice, stream));
      if (w.extended) TC_TRY(cudaMemcpyAsync(Zsnap, Zt, sizeof(float) * m * RHS, cudaMemcpyDeviceToDevice, stream));
    }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    TC_TRY(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t ce = cudaSuccess;
    for (int64_t q = 0; q < cnt && ce == cudaSuccess; ++q) {
      const int64_t k = k0 + q;
      ce = enqueue_iter(hplan[q], k, checking && (k % cfg->check_stride == 0 || k == cfg->max_iters));
    }
    cudaError_t ee = cudaStreamEndCapture(stream, &graph);
    if (ce != cudaSuccess || ee != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      snprintf(errbuf, errlen, "graph capture failed: %s", cudaGetErrorString(ce != cudaSuccess ? ce : ee));
      return -2;
    }
    TC_TRY(cudaGraphInstantiate(&gexec, graph, 0));
    TC_TRY(cudaGraphLaunch(gexec, stream));
    TC_TRY(cudaStreamSynchronize(stream));
    cudaGraphExecDestroy(gexec);
    cudaGraphDestroy(graph);
    if (checking) {
      int32_t nd = 0;
      TC_TRY(cudaMemcpyAsync(&nd, d_ndone, sizeof nd, cudaMemcpyDeviceToHost, stream));
      TC_TRY(cudaStreamSynchronize(stream));
      if (nd == R) {
        std::vector<int64_t> it(R);
        TC_TRY(cudaMemcpy(it.data(), d_iters, sizeof(int64_t) * R, cudaMemcpyDeviceToHost));
        K = *std::max_element(it.begin(), it.end());
        all_done = true;
        if (K < k0 + cnt - 1) {  // rewind to the chunk start and replay up to K exactly
          TC_TRY(cudaMemcpyAsync(Xt, Xsnap, sizeof(float) * n * RHS, cudaMemcpyDeviceToDevice, stream));
          if (w.extended) TC_TRY(cudaMemcpyAsync(Zt, Zsnap, sizeof(float) * m * RHS, cudaMemcpyDeviceToDevice, stream));
          for (int64_t k = k0; k <= K; ++k) TC_TRY(enqueue_iter(hplan[k - k0], k, false));
        }
      }
    }
  }
  TC_TRY(cudaEventRecord(ev1, stream));
  TC_TRY(cudaStreamSynchronize(stream));
  float ms = 0.f;
  TC_TRY(cudaEventElapsedTime(&ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  *loop_ms = ms;
  *k_final = K;
  // results back to the row-major layout of the caller
  k_from_t<<<dim3((unsigned)((n + 31) / 32), RHS / 32), tb, 0, stream>>>(Xt, n, n, R, w.X);
  if (w.extended) k_from_t<<<dim3((unsigned)((m + 31) / 32), RHS / 32), tb, 0, stream>>>(Zt, m, m, R, w.Z);
  TC_TRY(cudaGetLastError());
  if (iters_out) TC_TRY(cudaMemcpy(iters_out, d_iters, sizeof(int64_t) * R, cudaMemcpyDeviceToHost));
  if (errs_out) TC_TRY(cudaMemcpy(errs_out, d_errs_at, sizeof(double) * R, cudaMemcpyDeviceToHost));
  for (void* ptr : {(void*)Xt, (void*)Bt, (void*)Zt, (void*)Xst, (void*)Ut, (void*)Rt, (void*)part, (void*)Xsnap,
                    (void*)Zsnap, (void*)d_tol, (void*)d_errs_at, (void*)d_cpart, (void*)d_iters, (void*)d_ndone,
                    (void*)d_plan})
    if (ptr) cudaFreeAsync(ptr, stream);
  TC_TRY(cudaStreamSynchronize(stream));
  return 0;
}

}  // namespace rebk

// rebk_dense_split.cu — REBK with the column sweep and the row sweep on two
// CTA groups that run concurrently (dense fp64, sm_100a).
//
// In step_rebk (solvers.py:324-337) the z sequence never depends on x:
//   u_k = A_Jᵀ z_{k-1},  z_k = z_{k-1} - s_J A_J u_k          (column sweep)
//   r_k = A_I x_{k-1} - b_I + z_{k,I},  x_k = x_{k-1} - s_I A_Iᵀ r_k  (row sweep)
// The row sweep only needs the |I| entries z_{k,I}.  So clusters [0, ncc)
// run the column sweep (each CTA owns a slice of z rows), the other clusters
// run the row sweep (each CTA owns a slice of x columns), and the column
// group streams z_{k,I_k} one way to the row group through a ring of 16-byte
// {value, seq} words.  Each group has ONE grid-wide sum per iteration on its
// own critical path (the fused kernel had both in series); the column group
// runs up to D iterations ahead (flow control on the row group's progress)
// and keeps H >= D + 3 iterations of z history, so the run stops with the
// exact state (x_K, z_K) of the first converged check K.
//
// Exchanges, tiles and products are the fast path's (rebk_dense_fast.cu):
// TMA 2D tiles, DSMEM st.async + LL128 exchanges inside each group, fixed
// summation order (bitwise replay).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rebk_device.cuh"
#include "rebk_internal.h"

namespace rebk {

constexpr int kSplitThreads = 512;  // 4 warps per SM sub-partition: the tile products are latency-bound

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// The cluster shape is a kernel attribute (not a launch attribute), so the
// kernel always runs with its clusters, also when a profiler replays it
__global__ void __launch_bounds__(kSplitThreads, 1) __cluster_dims__(kClusterCS, 1, 1)
    rebk_dense_split_kernel(const __grid_constant__ SplitParams spp, const __grid_constant__ CUtensorMap tm_ct,
                            const __grid_constant__ CUtensorMap tm_rt) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t mbar[2];  // this CTA's tile (column or row): first / second row half
  __shared__ __align__(8) uint64_t xbar[2];  // exchange receive barriers: 0 scatter, 1 broadcast
  __shared__ double s_errp;
  __shared__ int s_flag;

  const FastParams& fp = spp.f;
  const DenseParams& p = fp.d;
  const int CS = (int)cooperative_groups::this_cluster().num_blocks();
  const int crank = (int)cooperative_groups::this_cluster().block_rank();
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int cid = g / CS, NC = G / CS;
  Control* ctl = p.ctl;
  SplitShared* sh = spp.sh;
  if (*((volatile int32_t*)&ctl->done)) return;
  if (CS != fp.cluster_size || G % CS != 0 || spp.ncc < 1 || spp.ncc >= NC) {
    if (tid == 0) atomicExch(&ctl->fault, 1);
    return;
  }
  const bool colgrp = cid < spp.ncc;
  const int NCg = colgrp ? spp.ncc : NC - spp.ncc;  // clusters in my group
  const int lcid = colgrp ? cid : cid - spp.ncc;    // my cluster within the group
  const int Gg = NCg * CS;                          // CTAs in my group
  const int gg = lcid * CS + crank;                 // my index within the group

  const int zr0 = split_rows(p.m, Gg, gg), zr1 = split_rows(p.m, Gg, gg + 1);  // column group
  const int xq0 = split_even(p.n, Gg, gg), xq1 = split_even(p.n, Gg, gg + 1);  // row group
  const int nR = colgrp ? zr1 - zr0 : 0, nC = colgrp ? 0 : xq1 - xq0;

  double* s_tile = sm;  // column tile (column group) or row tile (row group)
  // group-specific vector areas (split_geometry): the column group holds z,
  // the row group x and x*; s_cin (last) holds every cluster's partials
  double* base = sm + (colgrp ? spp.vec_off_c : spp.vec_off_r);
  double* s_z = base;
  double* s_x = base;
  double* s_xs = s_x + fp.pad_nC;
  double* s_u = colgrp ? s_z + fp.pad_nR : s_xs + fp.pad_nC;
  double* s_r = s_u + fp.pad_ne;
  double* s_part = s_r + fp.pad_ne;
  double* s_in = s_part + fp.pad_ne;
  double* s_red = s_in + fp.pad_in;
  double* s_cin = s_red + 2 * kSplitThreads;

  for (int c = tid; c < nC; c += kSplitThreads) {
    s_x[c] = __ldcg(p.x + xq0 + c);
    s_xs[c] = p.xs ? __ldg(p.xs + xq0 + c) : 0.0;
  }
  for (int r = tid; r < nR; r += kSplitThreads) s_z[r] = __ldcg(p.z + zr0 + r);
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
    prefetch_tensormap(colgrp ? &tm_ct : &tm_rt);
    s_errp = 0.0;
  }
  __syncthreads();
  uint32_t xpar[2] = {0u, 0u};
  cluster_sync_rel_acq();

  long long prof_acc[16];
  for (int i = 0; i < 16; ++i) prof_acc[i] = 0;
  long long prof_last = clock64();
#define PROF(i)                      \
  if (p.prof) {                      \
    const long long _t = clock64();  \
    prof_acc[i] += _t - prof_last;   \
    prof_last = _t;                  \
  }
  const int xb = colgrp ? 8 : 12;  // exchange-internal profile marks of my group
  // ---- group exchange (same protocol as the fast path, group-local)
  unsigned long long xseq = colgrp ? *((volatile unsigned long long*)&ctl->xseq)
                                   : *((volatile unsigned long long*)&ctl->xseq_row);
  LLWord* cpart_g = colgrp ? fp.cpart_u : fp.cpart_r;
  const int stride_g = colgrp ? fp.stride_u : fp.stride_r;
  const bool gather_all = (spp.xmode >> (colgrp ? 0 : 1)) & 1;
  int64_t cur_k = 0;  // iteration of the running exchange (REBK_TRACE)
  auto stamp = [&](int i) {
#ifdef REBK_SPLIT_TRACE  // tools/build_variants.sh trace "-DREBK_SPLIT_TRACE"
    if (spp.trace && tid == 0 && cur_k >= spp.trace_k0 && cur_k < spp.trace_k0 + spp.trace_n) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      spp.trace[((size_t)(cur_k - spp.trace_k0) * G + g) * 8 + i] = t;
    }
#else
    (void)i;
    (void)cur_k;
#endif
  };
  // pre(e) runs on the thread that will finalize entry e of this CTA's slice,
  // before the exchange waits on anything (e.g. a ring poll that is usually
  // already satisfied); its value is handed to finalize(e, sum, pre).
  auto exchange = [&](int ne, double* s_out, auto pre, auto finalize) {
    stamp(0);
    const unsigned long long seq = ++xseq;
    const int sl = (ne + CS - 1) / CS;
    const int e0 = crank * sl;
    const int e1 = (e0 + sl < ne) ? e0 + sl : ne;
    const int nmy = e1 > e0 ? e1 - e0 : 0;
    // two LL slots by sequence parity: a cluster can only reach exchange
    // seq+2 after every cluster has published seq+1, i.e. after every CTA has
    // finished reading the words of exchange seq
    LLWord* cslot = cpart_g + (seq & 1ull) * (size_t)NC * stride_g;
    if (tid == 0) mbar_arrive_expect_tx(&xbar[0], (uint32_t)(CS * nmy * 8));
    const uint32_t in_base = smem_u32(s_in), bar0 = smem_u32(&xbar[0]);
    for (int e = tid; e < ne; e += kSplitThreads) {
      const int dst = e / sl;
      st_async_f64(mapa_u32(in_base + 8u * (uint32_t)(crank * sl + (e - dst * sl)), dst), s_part[e],
                   mapa_u32(bar0, dst));
    }
    // slices are at most NT entries (ne <= 2 * 256 + 1 < CS * NT): one entry per thread
    const double2 mypre = tid < nmy ? pre(e0 + tid) : make_double2(0.0, 0.0);
    if (tid == 0) mbar_wait(&xbar[0], xpar[0]);
    xpar[0] ^= 1u;
    __syncthreads();
    stamp(1);
    PROF(xb + 0);
    if (NCg == 1) {
      // a group of ONE cluster (C1): the cluster sums are final, so the
      // round trip through the global LL words is skipped — slice owners
      // finalize and broadcast straight from the scattered partials
      // (0.0 + sum: the same value the one-term cluster sum would give)
      if (tid == 0) mbar_arrive_expect_tx(&xbar[1], (uint32_t)(ne * 8));
      __syncthreads();
      PROF(xb + 2);
      const uint32_t out_base = smem_u32(s_out), bar1 = smem_u32(&xbar[1]);
      for (int e = tid; e < nmy; e += kSplitThreads) {
        double acc = 0.0;
        for (int q = 0; q < CS; ++q) acc += s_in[q * sl + e];
        acc = finalize(e0 + e, 0.0 + acc, mypre);
        const uint32_t la = out_base + 8u * (uint32_t)(e0 + e);
        for (int dst = 0; dst < CS; ++dst) st_async_f64(mapa_u32(la, dst), acc, mapa_u32(bar1, dst));
      }
      if (tid == 0) mbar_wait(&xbar[1], xpar[1]);
      xpar[1] ^= 1u;
      __syncthreads();
      stamp(3);
      PROF(xb + 3);
      return;
    }
    for (int e = tid; e < nmy; e += kSplitThreads) {
      double acc = 0.0;
      for (int q = 0; q < CS; ++q) acc += s_in[q * sl + e];
      st_ll(cslot + (size_t)lcid * stride_g + e0 + e, acc, seq);
    }
    PROF(xb + 1);
    if (gather_all) {
      // every CTA gathers all clusters' partials for ALL entries and reduces
      // them itself (same fixed order over clusters): no broadcast step
      for (int t = tid; t < NCg * ne; t += kSplitThreads) {
        const int q = t / ne, e = t - q * ne;
        s_cin[t] = poll_ll(cslot + (size_t)q * stride_g + e, seq);
      }
      __syncthreads();
      PROF(xb + 2);
      for (int e = tid; e < ne; e += kSplitThreads) {
        double acc = 0.0;
        for (int q = 0; q < NCg; ++q) acc += s_cin[q * ne + e];
        s_out[e] = finalize(e, acc, pre(e));
      }
      __syncthreads();
    } else {
      // slice owners reduce their slice over clusters and broadcast it back
      // to the cluster peers by st.async
      for (int t = tid; t < NCg * nmy; t += kSplitThreads) {
        const int q = t / nmy, e = t - q * nmy;
        s_cin[t] = poll_ll(cslot + (size_t)q * stride_g + e0 + e, seq);
      }
      if (tid == 0) mbar_arrive_expect_tx(&xbar[1], (uint32_t)(ne * 8));
      __syncthreads();
      stamp(2);
      PROF(xb + 2);
      const uint32_t out_base = smem_u32(s_out), bar1 = smem_u32(&xbar[1]);
      for (int e = tid; e < nmy; e += kSplitThreads) {
        double acc = 0.0;
        for (int q = 0; q < NCg; ++q) acc += s_cin[q * nmy + e];
        acc = finalize(e0 + e, acc, mypre);
        const uint32_t la = out_base + 8u * (uint32_t)(e0 + e);
        for (int dst = 0; dst < CS; ++dst) st_async_f64(mapa_u32(la, dst), acc, mapa_u32(bar1, dst));
      }
      if (tid == 0) mbar_wait(&xbar[1], xpar[1]);
      xpar[1] ^= 1u;
      __syncthreads();
    }
    stamp(3);
    PROF(xb + 3);
  };
  auto ident = [](int, double s, double2) { return s; };
  auto nopre = [](int) { return make_double2(0.0, 0.0); };

  // The tile arrives as two half-height TMA boxes (rows [0, hb) and
  // [hb, 2hb)), each on its own mbarrier; both flip phase once per iteration.
  // A half's buffer is refilled with the next tile's half as soon as the
  // second product pass is done with it.
  const int hb = colgrp ? fp.ct_box_h : fp.rt_box_h;
  const int tw = colgrp ? fp.ct_box_w : fp.rt_box_w;
  const int hoff = (hb * tw + 15) & ~15;  // second half starts 128-byte aligned (TMA destination)
  double* s_tileB = s_tile + hoff;
  uint32_t tile_par = 0;
  bool in_flight[2] = {false, false};
  const bool two = spp.pieces == 2;
  auto wait_half = [&](int hf) {  // every thread waits itself
    if (hf == 1 && !two) return;
    mbar_wait(&mbar[hf], tile_par);
    in_flight[hf] = false;
  };
  auto issue_half = [&](const Plan& pl, int hf) {  // caller: all readers of this half are done
    if (hf == 1 && !two) return;
    in_flight[hf] = true;
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&mbar[hf], (uint32_t)(tw * hb * 8));
      if (colgrp)
        tma_load_2d(hf ? s_tileB : s_tile, &tm_ct, pl.c_lo, zr0 + hf * hb, &mbar[hf]);
      else
        tma_load_2d(hf ? s_tileB : s_tile, &tm_rt, xq0, pl.r_lo + hf * hb, &mbar[hf]);
    }
  };
  auto issue_tile = [&](const Plan& pl) {
    issue_half(pl, 0);
    issue_half(pl, 1);
  };
  auto nothing = []() {};
  // experiment switches (REBK_SPLIT_XMODE bits): 4 = issue both halves after
  // the second pass, 8 = one-row-per-thread rowdot2, 16 = rolled rowdot2x
  // (default: rowdot2u, measured fastest on C2: profiles/r01_split_variants.txt)
  const bool early_a = two && (spp.xmode & 4) == 0;  // refill the first half while the second is read
  const bool rd_old = (spp.xmode & 8) != 0;
  const bool rd_x = (spp.xmode & 16) != 0;
  auto rowdot = [&](const double* T, int R, int C, const double* v, auto epi) {
    if (rd_old)
      rowdot2<kSplitThreads>(T, tw, R, C, v, epi);
    else if (rd_x)
      rowdot2x<kSplitThreads>(T, tw, R, C, v, epi);
    else
      rowdot2u<kSplitThreads>(T, tw, R, C, v, epi);
  };

  if (colgrp) {
    // ================================ column sweep ================================
    const int D = spp.ring, H = spp.hist;
    int64_t k = p.k_begin;
    int64_t stopped_at = -1;  // K when the row group stopped the run
    if (p.k_begin <= p.k_end) issue_tile(p.plan[0]);
    Plan pl_next;
    if (p.k_begin <= p.k_end) pl_next = p.plan[0];
    for (; k <= p.k_end; ++k) {
      const Plan pl = pl_next;
      if (k < p.k_end) pl_next = p.plan[k + 1 - p.k_begin];
      const int nJ = pl.c_hi - pl.c_lo;
      cur_k = k;
      wait_half(0);
      // the next tile heads for L2 now; its TMA loads (during the z update)
      // then come from L2 instead of HBM
      if (tid == 0 && k < p.k_end) {
        tma_prefetch_l2_2d(&tm_ct, pl_next.c_lo, zr0);
        if (two) tma_prefetch_l2_2d(&tm_ct, pl_next.c_lo, zr0 + hb);
      }
      stamp(4);
      PROF(0);
      const int hA = nR < hb ? nR : hb;
      colsum2h<kSplitThreads>(
          s_tile, s_tileB, tw, nR, hA, nJ, s_z, s_red,
          [&]() {
            stamp(5);
            wait_half(1);
            stamp(6);
          },
          nothing,
          [&](int c, double val) { s_part[c] = val; });
      tile_par ^= 1u;
      // the stop flag rides the exchange so every column CTA leaves at the
      // same iteration (a CTA that left alone would strand the others in it)
      if (tid == 0) s_part[nJ] = ld_acquire_u64(&sh->stop) != 0 ? 1.0 : 0.0;
      __syncthreads();
      PROF(1);
      exchange(nJ + 1, s_u, nopre, ident);
      if (s_u[nJ] != 0.0) break;
      const double cs = pl.c_scale;
      double* hist = spp.zhist + (size_t)(k % H) * p.m;
      auto zupd = [&](int r, double acc) {
        const double zn = s_z[r] - cs * acc;
        s_z[r] = zn;
        __stcg(hist + zr0 + r, zn);
      };
      rowdot(s_tile, hA, nJ, s_u, zupd);
      if (early_a) {
        __syncthreads();
        if (k < p.k_end) issue_half(pl_next, 0);
      }
      rowdot(s_tileB, nR - hA, nJ, s_u, [&](int r, double acc) { zupd(hA + r, acc); });
      __syncthreads();
      if (k < p.k_end) {
        if (!early_a) issue_half(pl_next, 0);
        issue_half(pl_next, 1);
      }
      stamp(7);
      PROF(2);
      // publish z_{k, I_k ∩ my rows}: wait until the ring slot is free
      const int lo = pl.r_lo > zr0 ? pl.r_lo : zr0, hi = pl.r_hi < zr1 ? pl.r_hi : zr1;
      if (lo < hi) {
        if (tid == 0) {
          while (true) {
            const unsigned long long prog = ld_acquire_u64(&sh->row_progress);
            if ((int64_t)prog + D >= k) {
              s_flag = 0;
              break;
            }
            if (ld_acquire_u64(&sh->stop) != 0) {
              s_flag = 1;
              break;
            }
          }
        }
        __syncthreads();
        if (!s_flag) {  // after a stop nobody reads the ring: skip, leave at the next exchange
          LLWord* slot = spp.zring + (size_t)(k % D) * spp.zr_stride;
          for (int i = lo + tid; i < hi; i += kSplitThreads)
            st_ll(slot + (i - pl.r_lo), s_z[i - zr0], (unsigned long long)k);
        }
      }
      PROF(3);
    }
    // the state to leave in global z: z_K if the row group stopped at K,
    // else the last iteration of this launch.  Wait for the row group's
    // verdict on this chunk first.
    if (tid == 0) {
      unsigned long long st;
      while (true) {
        st = ld_acquire_u64(&sh->stop);
        if (st != 0) break;
        if ((int64_t)ld_acquire_u64(&sh->row_progress) >= p.k_end) break;
      }
      s_flag = (int)st;  // K + 1 or 0
    }
    __syncthreads();
    const int64_t last = k - 1;  // last iteration computed here
    if (s_flag) {
      stopped_at = (int64_t)s_flag - 1;
      if (stopped_at < last && stopped_at >= p.k_begin) {
        const double* hist = spp.zhist + (size_t)(stopped_at % H) * p.m;
        for (int r = tid; r < nR; r += kSplitThreads) s_z[r] = __ldcg(hist + zr0 + r);
      } else if (stopped_at < p.k_begin) {
        for (int r = tid; r < nR; r += kSplitThreads) s_z[r] = __ldcg(p.z + zr0 + r);
      }
      __syncthreads();
    }
    for (int r = tid; r < nR; r += kSplitThreads) __stcg(p.z + zr0 + r, s_z[r]);
    if (g == 0 && tid == 0) ctl->xseq = xseq;
  } else {
    // ================================= row sweep ==================================
    const int D = spp.ring;
    const bool checking = p.stop_mode == 0;
    // Σ (x - x*)^2 over my columns by warp 0 alone (fixed order); s_errp is
    // read only by thread 0, so no block barrier is needed
    auto err_partial = [&]() {
      if (tid < 32) {
        double acc = 0.0;
        for (int c = tid; c < nC; c += 32) {
          const double d = s_x[c] - s_xs[c];
          acc = fma(d, d, acc);
        }
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (tid == 0) s_errp = acc;
      }
    };
    const bool leader = (gg == 0 && tid == 0);
    auto decide = [&](double sumsq, int64_t k) -> bool {
      const double err = sqrt(sumsq);
      const bool conv = check_stops(err, p.tol, p.nonfinite_stop);
      if (leader) {
        record_check(ctl, p.errs, p.errs_cap, p.record, err, p.tol, p.nonfinite_stop, k);
        if (conv) st_release_u64(&sh->stop, (unsigned long long)k + 1);
      }
      return conv;
    };
    auto solo_check = [&](int64_t k) -> bool {
      if (tid == 0) s_part[0] = s_errp;
      __syncthreads();
      exchange(1, s_r, nopre, ident);
      return decide(s_r[0], k);
    };
    bool finished = false;
    if (p.k_begin == 1 && checking) {
      err_partial();
      if (solo_check(0)) finished = true;
    }
    bool pending = false;
    int64_t pending_k = 0;
    int64_t k = p.k_begin;
    if (!finished && p.k_begin <= p.k_end) issue_tile(p.plan[0]);
    Plan pl_next;
    if (p.k_begin <= p.k_end) pl_next = p.plan[0];
    for (; !finished && k <= p.k_end; ++k) {
      const Plan pl = pl_next;
      if (k < p.k_end) pl_next = p.plan[k + 1 - p.k_begin];
      const int nI = pl.r_hi - pl.r_lo;
      cur_k = k;
      const bool check_k = checking && (k % p.stride == 0);
      wait_half(0);
      if (tid == 0 && k < p.k_end) {
        tma_prefetch_l2_2d(&tm_rt, xq0, pl_next.r_lo);
        if (two) tma_prefetch_l2_2d(&tm_rt, xq0, pl_next.r_lo + hb);
      }
      stamp(4);
      PROF(4);
      const int hA = nI < hb ? nI : hb;
      rowdot(s_tile, hA, nC, s_x, [&](int r, double acc) { s_part[r] = acc; });
      stamp(5);
      wait_half(1);
      stamp(6);
      rowdot(s_tileB, nI - hA, nC, s_x,
                             [&](int r, double acc) { s_part[hA + r] = acc; });
      tile_par ^= 1u;
      if (pending && tid == 0) s_part[nI] = s_errp;
      __syncthreads();
      PROF(5);
      const int rl = pl.r_lo;
      const LLWord* slot = spp.zring + (size_t)(k % D) * spp.zr_stride;
      // r = ((Σ_g rpart) - b_I) + z_{k,I}; z_{k,I} arrives from the column group
      // pre: {b_e, z_{k,e}} are fetched while the partial sums travel
      auto bz = [&](int e) {
        if (e >= nI) return make_double2(0.0, 0.0);
        return make_double2(__ldg(p.b + rl + e), p.extended ? poll_ll(slot + e, (unsigned long long)k) : 0.0);
      };
      exchange(nI + (pending ? 1 : 0), s_r, bz, [&](int e, double s, double2 pz) {
        if (e >= nI) return s;
        double rv = s - pz.x;
        if (p.extended) rv += pz.y;
        return rv;
      });
      if (pending) {
        pending = false;
        if (decide(s_r[nI], pending_k)) {  // sets sh->stop before any progress past k-1 is visible
          finished = true;
          break;
        }
      }
      if (leader) st_release_u64(&sh->row_progress, (unsigned long long)k);
      const double rs = pl.r_scale;
      colsum2h<kSplitThreads, true>(
          s_tile, s_tileB, tw, nI, hA, nC, s_r, s_red,
          [&]() {
            if (early_a) {
              __syncthreads();
              if (k < p.k_end) issue_half(pl_next, 0);
            }
          },
          [&]() {
            __syncthreads();
            if (k < p.k_end) {
              if (!early_a) issue_half(pl_next, 0);
              issue_half(pl_next, 1);
            }
          },
          [&](int c, double acc) { s_x[c] = s_x[c] - rs * acc; });
      stamp(7);
      if (check_k) {
        err_partial();
        pending = true;
        pending_k = k;
      }
      PROF(6);
    }
    if (!finished) {
      if (pending) {
        if (solo_check(pending_k)) finished = true;
      }
      if (!finished && p.k_end == p.max_iters) {
        if (checking && (p.max_iters % p.stride) != 0) {
          err_partial();
          solo_check(p.max_iters);
        }
        if (leader) {
          if (!ctl->converged) ctl->iters = p.max_iters;
          ctl->done = 1;
        }
      }
    }
    for (int c = tid; c < nC; c += kSplitThreads) __stcg(p.x + xq0 + c, s_x[c]);
    if (leader) ctl->xseq_row = xseq;
  }
  if (p.prof && tid == 0)
    for (int i = 0; i < 16; ++i) p.prof[g * 16 + i] = prof_acc[i];
#undef PROF
  // no TMA may still be writing into shared memory when the CTA exits
  if (in_flight[0]) wait_half(0);
  if (in_flight[1]) wait_half(1);
  __syncthreads();
  cluster_sync_rel_acq();
}

static cudaError_t set_split_attrs() {
  static int configured_device = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured_device == dev) return cudaSuccess;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(rebk_dense_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(rebk_dense_split_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  configured_device = dev;
  return cudaSuccess;
}

cudaError_t launch_dense_split(const SplitParams& sp, const CUtensorMap& tm_ct, const CUtensorMap& tm_rt, int G,
                               int cluster_size, size_t smem_bytes, cudaStream_t stream) {
  cudaError_t e = set_split_attrs();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kSplitThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  if (cluster_size != kClusterCS) return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, rebk_dense_split_kernel, sp, tm_ct, tm_rt);
}

cudaError_t split_max_clusters(int cluster_size, size_t smem_bytes, int* clusters) {
  cudaError_t e = set_split_attrs();
  if (e != cudaSuccess) return e;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((sms / cluster_size) * cluster_size);
  cfg.blockDim = dim3(kSplitThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_size;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(clusters, (void*)rebk_dense_split_kernel, &cfg);
}

}  // namespace rebk

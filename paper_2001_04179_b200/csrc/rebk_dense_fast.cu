// rebk_dense_fast.cu — clustered persistent fp64 REBK kernel (the fast path).
//
// Same iteration and ownership as rebk_dense.cu (step_rebk, solvers.py:324-337;
// CTA g owns z rows [zr0, zr1) and x columns [xq0, xq1)), re-organised around
// what the B200 measurements showed dominates:
//   * each block tile arrives with ONE 2D TMA copy (cp.async.bulk.tensor)
//     instead of one bulk copy per row;
//   * the four tile products read shared memory as 16-byte pairs with
//     independent accumulator chains (latency-tolerant, conflict-free);
//   * each grid-wide sum (u = A_JᵀZ, r = A_I x - b_I + z_I) is ONE exchange
//     with no grid barrier at all:
//       - partial slices go to the slice-owning cluster peer by DSMEM st.async,
//         counted on the receiver's mbarrier (no cluster barrier, no membar);
//       - each slice owner publishes its cluster sum as a 16-byte {value,
//         seq} word (one STG.128); every consumer polls the words it needs
//         (LL128-style: data and flag arrive in the same store);
//       - slice totals are broadcast back to the cluster peers by st.async.
//     z_I rides inside the r exchange (exact: one non-zero contribution), so
//     no CTA ever reads another CTA's state through L2.
//     Fixed summation order everywhere, so runs replay bit for bit.
// Measured on B200: grid barrier 1.2 us, cluster barrier with
// its GPU-scope membar ~0.4 us; this exchange avoids both.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rebk_device.cuh"
#include "rebk_internal.h"

namespace cg = cooperative_groups;

namespace rebk {


__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(kClusterCS, 1, 1)
    rebk_dense_fast_kernel(const __grid_constant__ FastParams fp, const __grid_constant__ CUtensorMap tm_ct,
                           const __grid_constant__ CUtensorMap tm_rt) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t mbar[2];  // 0: column tile, 1: row tile
  __shared__ __align__(8) uint64_t xbar[2];  // exchange receive barriers: 0 scatter, 1 broadcast
  __shared__ double s_errp;                  // this CTA's pending error partial

  const DenseParams& p = fp.d;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int cid = g / CS, NC = G / CS;
  Control* ctl = p.ctl;
  if (*((volatile int32_t*)&ctl->done)) return;
  if (CS != fp.cluster_size || G % CS != 0) {  // launched without the expected clusters
    if (tid == 0) atomicExch(&ctl->fault, 1);
    return;
  }

  const int zr0 = split_rows(p.m, G, g), zr1 = split_rows(p.m, G, g + 1);
  const int xq0 = split_even(p.n, G, g), xq1 = split_even(p.n, G, g + 1);
  const int nR = zr1 - zr0, nC = xq1 - xq0;

  double* s_ct = sm + p.ct_off;
  double* s_rt = sm + p.rt_off;
  double* s_x = sm + p.vec_off;  // all vectors 16-byte aligned (even offsets)
  double* s_xs = s_x + fp.pad_nC;
  double* s_z = s_xs + fp.pad_nC;
  double* s_u = s_z + fp.pad_nR;
  double* s_r = s_u + fp.pad_ne;
  double* s_part = s_r + fp.pad_ne;
  double* s_in = s_part + fp.pad_ne;     // [CS][slice]
  double* s_cin = s_in + fp.pad_in;      // [NC][slice]
  double* s_red = s_cin + fp.pad_cin;    // 2 * kThreads

  for (int c = tid; c < nC; c += kThreads) {
    s_x[c] = __ldcg(p.x + xq0 + c);
    s_xs[c] = p.xs ? __ldg(p.xs + xq0 + c) : 0.0;
  }
  if (p.extended)
    for (int r = tid; r < nR; r += kThreads) s_z[r] = __ldcg(p.z + zr0 + r);
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
    prefetch_tensormap(&tm_ct);
    prefetch_tensormap(&tm_rt);
    s_errp = 0.0;
  }
  __syncthreads();
  uint32_t xpar[2] = {0u, 0u};
  cluster_sync_rel_acq();  // peers' exchange barriers are initialised before any st.async

  long long prof_acc[16];
  for (int i = 0; i < 16; ++i) prof_acc[i] = 0;
  long long prof_last = clock64();
#define PROF(i)                                  \
  if (p.prof) {                                  \
    const long long _t = clock64();              \
    prof_acc[i] += _t - prof_last;               \
    prof_last = _t;                              \
  }
  // One grid-wide sum of the ne-entry partial vectors s_part of every CTA;
  // the result (after finalize) lands in s_out of every CTA.  No grid
  // barrier: inside a cluster the partial slices travel by DSMEM st.async
  // (completion counted on the receiver's mbarrier); across clusters each
  // slice owner publishes {value, seq} 16-byte words that the consumers poll.
  unsigned long long xseq = *((volatile unsigned long long*)&ctl->xseq);
  auto exchange = [&](int ne, LLWord* cpart, int stride, double* s_out, auto finalize) {
    const unsigned long long seq = ++xseq;
    const int sl = (ne + CS - 1) / CS;
    const int e0 = crank * sl;
    const int e1 = (e0 + sl < ne) ? e0 + sl : ne;
    const int nmy = e1 > e0 ? e1 - e0 : 0;
    cpart += (seq & 1ull) * (size_t)NC * stride;  // two LL slots by sequence parity
    if (tid == 0) mbar_arrive_expect_tx(&xbar[0], (uint32_t)(CS * nmy * 8));
    const uint32_t in_base = smem_u32(s_in), bar0 = smem_u32(&xbar[0]);
    for (int e = tid; e < ne; e += kThreads) {
      const int dst = e / sl;
      st_async_f64(mapa_u32(in_base + 8u * (uint32_t)(crank * sl + (e - dst * sl)), dst), s_part[e],
                   mapa_u32(bar0, dst));
    }
    if (tid == 0) mbar_wait(&xbar[0], xpar[0]);
    xpar[0] ^= 1u;
    __syncthreads();
    PROF(10);
    for (int e = tid; e < nmy; e += kThreads) {
      double acc = 0.0;
      for (int q = 0; q < CS; ++q) acc += s_in[q * sl + e];
      st_ll(cpart + (size_t)cid * stride + e0 + e, acc, seq);
    }
    PROF(11);
    for (int t = tid; t < NC * nmy; t += kThreads) {
      const int q = t / nmy, e = t - q * nmy;
      s_cin[t] = poll_ll(cpart + (size_t)q * stride + e0 + e, seq);
    }
    if (tid == 0) mbar_arrive_expect_tx(&xbar[1], (uint32_t)(ne * 8));
    __syncthreads();
    PROF(12);
    const uint32_t out_base = smem_u32(s_out), bar1 = smem_u32(&xbar[1]);
    for (int e = tid; e < nmy; e += kThreads) {
      double acc = 0.0;
      for (int q = 0; q < NC; ++q) acc += s_cin[q * nmy + e];
      acc = finalize(e0 + e, acc);
      const uint32_t la = out_base + 8u * (uint32_t)(e0 + e);
      for (int dst = 0; dst < CS; ++dst) st_async_f64(mapa_u32(la, dst), acc, mapa_u32(bar1, dst));
    }
    PROF(13);
    if (tid == 0) mbar_wait(&xbar[1], xpar[1]);
    xpar[1] ^= 1u;
    __syncthreads();
    PROF(14);
  };
  auto ident = [](int, double s) { return s; };

  auto err_partial = [&]() {
    double acc = 0.0;
    for (int c = tid; c < nC; c += kThreads) {
      const double d = s_x[c] - s_xs[c];
      acc = fma(d, d, acc);
    }
    const double s = block_sum(acc, s_red);
    if (tid == 0) s_errp = s;
    __syncthreads();
  };
  auto decide = [&](double sumsq, int64_t k) -> bool {
    const double err = sqrt(sumsq);
    const bool conv = check_stops(err, p.tol, p.nonfinite_stop);
    if (g == 0 && tid == 0) record_check(ctl, p.errs, p.errs_cap, p.record, err, p.tol, p.nonfinite_stop, k);
    return conv;
  };
  // a stand-alone error exchange (check(0), end-of-chunk, off-stride final check)
  auto solo_check = [&](int64_t k) -> bool {
    if (tid == 0) s_part[0] = s_errp;
    __syncthreads();
    exchange(1, fp.cpart_u, fp.stride_u, s_u, ident);
    return decide(s_u[0], k);
  };

  bool ct_pending = false, rt_pending = false;
  uint32_t ct_par = 0, rt_par = 0;
  // one thread polls the mbarrier, the CTA barrier releases the others
  // (waiters parked in try_wait resume late; measured on B200)
  auto wait_ct = [&]() {
    if (ct_pending) {
#ifdef REBK_ALL_WAIT
      mbar_wait(&mbar[0], ct_par);
#else
      if (tid == 0) mbar_wait(&mbar[0], ct_par);
      __syncthreads();
#endif
      ct_par ^= 1u;
      ct_pending = false;
    }
  };
  auto wait_rt = [&]() {
    if (rt_pending) {
#ifdef REBK_ALL_WAIT
      mbar_wait(&mbar[1], rt_par);
#else
      if (tid == 0) mbar_wait(&mbar[1], rt_par);
      __syncthreads();
#endif
      rt_par ^= 1u;
      rt_pending = false;
    }
  };
  // the caller guarantees every thread finished reading the buffer (a barrier)
  auto issue_ct = [&](const Plan& pl) {
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&mbar[0], (uint32_t)(fp.ct_box_w * fp.ct_box_h * 8));
      tma_load_2d(s_ct, &tm_ct, pl.c_lo, zr0, &mbar[0]);
    }
    ct_pending = true;
  };
  auto issue_rt = [&](const Plan& pl) {
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&mbar[1], (uint32_t)(fp.rt_box_w * fp.rt_box_h * 8));
      tma_load_2d(s_rt, &tm_rt, xq0, pl.r_lo, &mbar[1]);
    }
    rt_pending = true;
  };


  const bool checking = p.stop_mode == 0;  // the fast path serves oracle_error / max_iters_only
  bool finished = false;
  if (p.k_begin == 1 && checking) {
    err_partial();
    if (solo_check(0)) finished = true;
  }
  bool pending = false;
  int64_t pending_k = 0;
  int64_t k = p.k_begin;
  if (!finished && p.extended && p.k_begin <= p.k_end) issue_ct(p.plan[0]);

  Plan pl_next;
  if (p.k_begin <= p.k_end) pl_next = p.plan[0];
  for (; !finished && k <= p.k_end; ++k) {
    const Plan pl = pl_next;  // loaded one iteration ahead (hides the L2 round trip)
    if (k < p.k_end) pl_next = p.plan[k + 1 - p.k_begin];
    const int nJ = pl.c_hi - pl.c_lo;
    const int nI = pl.r_hi - pl.r_lo;
    const bool check_k = checking && (k % p.stride == 0);

    __syncthreads();  // every reader of the row tile (previous x update) is done
    issue_rt(pl);
    PROF(0);

    if (p.extended) {
      // P1: partial u over the owned rows (+ the pending error partial)
      wait_ct();
      PROF(1);
      colsum2(s_ct, fp.ct_box_w, nR, nJ, s_z, s_red, [&](int c, double val) { s_part[c] = val; });
#ifdef REBK_ICACHE_EXPERIMENT
      PROF(15);
      colsum2(s_ct, fp.ct_box_w, nR, nJ, s_z, s_red, [&](int c, double val) { s_part[c] = val; });
#endif
      const int ne = nJ + (pending ? 1 : 0);
      if (pending && tid == 0) s_part[nJ] = s_errp;
      __syncthreads();
      PROF(2);
      exchange(ne, fp.cpart_u, fp.stride_u, s_u, ident);
      PROF(3);
      if (pending) {
        pending = false;
        if (decide(s_u[nJ], pending_k)) {
          finished = true;
          break;
        }
      }
      // P3a: z[owned rows] -= s_J · A[rows, J] u ; then the column tile is free
      const double cs = pl.c_scale;
      rowdot2(s_ct, fp.ct_box_w, nR, nJ, s_u, [&](int r, double acc) {
        const double zn = s_z[r] - cs * acc;
        s_z[r] = zn;
        __stcg(p.z + zr0 + r, zn);
      });
      __syncthreads();
      if (k < p.k_end) issue_ct(pl_next);
      PROF(4);
    }
    // P3b: partial r over the owned columns
    wait_rt();
    PROF(5);
    rowdot2(s_rt, fp.rt_box_w, nI, nC, s_x, [&](int r, double acc) { s_part[r] = acc; });
    // entries [nI, 2 nI): z_I from the owning CTAs (zeros elsewhere, so the
    // sum is exact) -- it travels with the exchange instead of through L2
    const int nz = p.extended ? nI : 0;
    const int rl = pl.r_lo;
    for (int e = tid; e < nz; e += kThreads) {
      const int row = rl + e;
      s_part[nI + e] = (row >= zr0 && row < zr1) ? s_z[row - zr0] : 0.0;
    }
    const bool row_err = !p.extended && pending;
    if (row_err && tid == 0) s_part[nI + nz] = s_errp;
    __syncthreads();
    PROF(6);
    // P4: r = ((Σ_g rpart) - b_I) + z_I
    exchange(nI + nz + (row_err ? 1 : 0), fp.cpart_r, fp.stride_r, s_r, [&](int e, double s) { return s; });
    // r = ((Σ_g rpart) - b_I) + z_I  (solvers.py:291-294 order)
    for (int e = tid; e < nI; e += kThreads) {
      double rv = s_r[e] - __ldg(p.b + rl + e);
      if (p.extended) rv += s_r[nI + e];
      s_r[e] = rv;
    }
    __syncthreads();
    PROF(7);
    if (row_err) {
      pending = false;
      if (decide(s_r[nI + nz], pending_k)) {
        finished = true;
        break;
      }
    }
    // P5: x[owned cols] -= s_I · A[I, cols]ᵀ r
    const double rs = pl.r_scale;
    colsum2(s_rt, fp.rt_box_w, nI, nC, s_r, s_red, [&](int c, double acc) { s_x[c] = s_x[c] - rs * acc; });
    PROF(8);
    if (check_k) {
      err_partial();
      pending = true;
      pending_k = k;
    }
    PROF(9);
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
      if (g == 0 && tid == 0) {
        if (!ctl->converged) ctl->iters = p.max_iters;
        ctl->done = 1;
      }
    }
  }
  if (p.prof && tid == 0)
    for (int i = 0; i < 16; ++i) p.prof[g * 16 + i] = prof_acc[i];
  if (g == 0 && tid == 0) ctl->xseq = xseq;
#undef PROF
  for (int c = tid; c < nC; c += kThreads) __stcg(p.x + xq0 + c, s_x[c]);
  wait_ct();  // all threads: the waits contain a CTA barrier
  wait_rt();
  __syncthreads();
  cluster_sync_rel_acq();  // no CTA leaves while a peer may still write its shared memory
}

static cudaError_t set_fast_attrs() {
  static int configured_device = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured_device == dev) return cudaSuccess;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(rebk_dense_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(rebk_dense_fast_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  configured_device = dev;
  return cudaSuccess;
}

cudaError_t fast_max_clusters(int cluster_size, size_t smem_bytes, int* clusters) {
  cudaError_t e = set_fast_attrs();
  if (e != cudaSuccess) return e;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((sms / cluster_size) * cluster_size);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_size;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(clusters, (void*)rebk_dense_fast_kernel, &cfg);
}

cudaError_t launch_dense_fast(const FastParams& fp, const CUtensorMap& tm_ct, const CUtensorMap& tm_rt, int G,
                              int cluster_size, size_t smem_bytes, cudaStream_t stream) {
  cudaError_t e = set_fast_attrs();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  if (cluster_size != kClusterCS) return cudaErrorInvalidValue;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, rebk_dense_fast_kernel, fp, tm_ct, tm_rt);
}

}  // namespace rebk

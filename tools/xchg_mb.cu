// xchg_mb.cu — the split kernel's group exchange in isolation.
// 15 clusters of 8 CTAs (512 threads), groups of ncc and 15-ncc clusters,
// each CTA loops: spin `work` cycles, exchange ne entries (the split
// kernel's protocol: DSMEM scatter, LL publish/poll, DSMEM broadcast or
// gather-all).  Prints per-exchange microseconds per group and per mark.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2001_04179_b200/csrc xchg_mb.cu -o xchg_mb
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "rebk_device.cuh"
#include "rebk_internal.h"

using namespace rebk;
constexpr int NT = 512;

struct MbParams {
  int ncc, ne, iters, work, gather_all;
  LLWord* cpart;
  int stride;
  long long* prof;  // [G][8]
  double* out;
};

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(NT, 1) xchg_kernel(MbParams P) {
  __shared__ __align__(8) uint64_t xbar[2];
  __shared__ double s_part[512], s_out[512], s_in[512], s_cin[4096];
  const int CS = (int)cooperative_groups::this_cluster().num_blocks();
  const int crank = (int)cooperative_groups::this_cluster().block_rank();
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int cid = g / CS, NC = G / CS;
  const bool colgrp = cid < P.ncc;
  const int NCg = colgrp ? P.ncc : NC - P.ncc;
  const int lcid = colgrp ? cid : cid - P.ncc;
  LLWord* cpart_g = P.cpart + (colgrp ? 0 : (size_t)2 * NC * P.stride);
  if (tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  cluster_sync_rel_acq();
  uint32_t xpar[2] = {0u, 0u};
  long long acc_p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long last = clock64();
#define MK(i)                        \
  {                                  \
    const long long _t = clock64();  \
    acc_p[i] += _t - last;           \
    last = _t;                       \
  }
  unsigned long long xseq = 0;
  const int ne = P.ne;
  double chk = 0.0;
  for (int it = 0; it < P.iters; ++it) {
    // "products"
    if (P.work > 0) {
      const long long t0 = clock64();
      while (clock64() - t0 < P.work) {
      }
    }
    for (int e = tid; e < ne; e += NT) s_part[e] = (double)(g + e + it);
    __syncthreads();
    MK(0);
    const unsigned long long seq = ++xseq;
    const int sl = (ne + CS - 1) / CS;
    const int e0 = crank * sl;
    const int e1 = (e0 + sl < ne) ? e0 + sl : ne;
    const int nmy = e1 > e0 ? e1 - e0 : 0;
    LLWord* cslot = cpart_g + (seq & 1ull) * (size_t)NC * P.stride;
    if (tid == 0) mbar_arrive_expect_tx(&xbar[0], (uint32_t)(CS * nmy * 8));
    const uint32_t in_base = smem_u32(s_in), bar0 = smem_u32(&xbar[0]);
    for (int e = tid; e < ne; e += NT) {
      const int dst = e / sl;
      st_async_f64(mapa_u32(in_base + 8u * (uint32_t)(crank * sl + (e - dst * sl)), dst), s_part[e],
                   mapa_u32(bar0, dst));
    }
    if (tid == 0) mbar_wait(&xbar[0], xpar[0]);
    xpar[0] ^= 1u;
    __syncthreads();
    MK(1);
    for (int e = tid; e < nmy; e += NT) {
      double acc = 0.0;
      for (int q = 0; q < CS; ++q) acc += s_in[q * sl + e];
      st_ll(cslot + (size_t)lcid * P.stride + e0 + e, acc, seq);
    }
    MK(2);
    if (P.gather_all) {
      for (int t = tid; t < NCg * ne; t += NT) {
        const int q = t / ne, e = t - q * ne;
        s_cin[t] = poll_ll(cslot + (size_t)q * P.stride + e, seq);
      }
      __syncthreads();
      MK(3);
      for (int e = tid; e < ne; e += NT) {
        double acc = 0.0;
        for (int q = 0; q < NCg; ++q) acc += s_cin[q * ne + e];
        s_out[e] = acc;
      }
      __syncthreads();
    } else {
      for (int t = tid; t < NCg * nmy; t += NT) {
        const int q = t / nmy, e = t - q * nmy;
        s_cin[t] = poll_ll(cslot + (size_t)q * P.stride + e0 + e, seq);
      }
      if (tid == 0) mbar_arrive_expect_tx(&xbar[1], (uint32_t)(ne * 8));
      __syncthreads();
      MK(3);
      const uint32_t out_base = smem_u32(s_out), bar1 = smem_u32(&xbar[1]);
      for (int e = tid; e < nmy; e += NT) {
        double acc = 0.0;
        for (int q = 0; q < NCg; ++q) acc += s_cin[q * nmy + e];
        const uint32_t la = out_base + 8u * (uint32_t)(e0 + e);
        for (int dst = 0; dst < CS; ++dst) st_async_f64(mapa_u32(la, dst), acc, mapa_u32(bar1, dst));
      }
      if (tid == 0) mbar_wait(&xbar[1], xpar[1]);
      xpar[1] ^= 1u;
      __syncthreads();
    }
    MK(4);
    chk += s_out[(it * 7) % ne];
  }
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) P.prof[g * 8 + i] = acc_p[i];
    P.out[g] = chk;
  }
}

int main(int argc, char** argv) {
  const int ncc = argc > 1 ? atoi(argv[1]) : 4;
  const int ne = argc > 2 ? atoi(argv[2]) : 201;
  const int work = argc > 3 ? atoi(argv[3]) : 0;
  const int gather = argc > 4 ? atoi(argv[4]) : 0;
  const int iters = 20000, G = 120, NC = 15;
  MbParams P{ncc, ne, iters, work, gather, nullptr, 512, nullptr, nullptr};
  cudaMalloc(&P.cpart, 4 * (size_t)NC * P.stride * sizeof(LLWord));
  cudaMemset(P.cpart, 0, 4 * (size_t)NC * P.stride * sizeof(LLWord));
  cudaMalloc(&P.prof, G * 8 * sizeof(long long));
  cudaMalloc(&P.out, G * sizeof(double));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  xchg_kernel<<<G, NT>>>(P);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[G * 8];
  cudaMemcpy(h, P.prof, sizeof h, cudaMemcpyDeviceToHost);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  printf("ncc=%d ne=%d work=%d gather=%d: %.3f us/iter total\n", ncc, ne, work, gather, 1e3 * ms / iters);
  for (int grp = 0; grp < 2; ++grp) {
    const int q0 = grp ? ncc * 8 : 0, q1 = grp ? G : ncc * 8;
    printf("  %s group (%d CTAs):", grp ? "row" : "col", q1 - q0);
    for (int i = 0; i < 5; ++i) {
      double m = 0;
      for (int q = q0; q < q1; ++q) m += (double)h[q * 8 + i] / (khz * 1e-3) / iters / (q1 - q0);
      printf(" m%d=%.3f", i, m);
    }
    printf("\n");
  }
  return 0;
}

// hop_mb.cu — one-way latency of the two exchange "hops": an LL128 word
// through L2 (ping-pong between two CTAs) and a DSMEM st.async inside a
// cluster (ping-pong between two CTAs of a cluster).  Not product code.
#include <cstdio>
#include "../paper_2001_04179_b200/csrc/rebk_device.cuh"
using namespace rebk;

__global__ void ll_pingpong(LLWord* w, int iters, long long* out) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;  // 0 or 1 (launched with gridDim 2 .. far apart SMs)
  if (me > 1) return;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (me == 0) { st_ll(w, 1.0, (unsigned long long)i); poll_ll(w + 1, (unsigned long long)i); }
    else { poll_ll(w, (unsigned long long)i); st_ll(w + 1, 2.0, (unsigned long long)i); }
  }
  long long t1 = clock64();
  if (me == 0) out[0] = (t1 - t0) / iters;
}

__global__ void __cluster_dims__(2, 1, 1) dsmem_pingpong(int iters, long long* out) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) double slot;
  const int rank = (int)cooperative_groups::this_cluster().block_rank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  cluster_sync_rel_acq();
  const uint32_t peer_slot = mapa_u32(smem_u32(&slot), rank ^ 1), peer_bar = mapa_u32(smem_u32(&bar), rank ^ 1);
  uint32_t par = 0;
  long long t0 = clock64();
  if (threadIdx.x == 0)
  for (int i = 0; i < iters; ++i) {
    if (rank == 0) {
      mbar_arrive_expect_tx(&bar, 8);
      st_async_f64(peer_slot, (double)i, peer_bar);
      mbar_wait(&bar, par); par ^= 1;
    } else {
      mbar_arrive_expect_tx(&bar, 8);
      mbar_wait(&bar, par); par ^= 1;
      st_async_f64(peer_slot, (double)i, peer_bar);
    }
  }
  long long t1 = clock64();
  if (rank == 0 && threadIdx.x == 0) out[1] = (t1 - t0) / iters;
  __syncwarp();
  cluster_sync_rel_acq();
}

int main() {
  LLWord* w; long long* d; cudaMalloc(&w, 64); cudaMalloc(&d, 64); cudaMemset(w, 0, 64);
  ll_pingpong<<<148, 32>>>(w, 20000, d);
  dsmem_pingpong<<<2, 32>>>(20000, d);
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  printf("LL128 word through L2: round trip %lld cycles = %.3f us, one way %.3f us\n", h[0], h[0] / (khz * 1e-3), h[0] / (khz * 1e-3) / 2);
  printf("DSMEM st.async + mbarrier: round trip %lld cycles = %.3f us, one way %.3f us\n", h[1], h[1] / (khz * 1e-3), h[1] / (khz * 1e-3) / 2);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

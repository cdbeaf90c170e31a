// rebk_csr_build.cu — the sparse context's derived arrays, built on the
// device from the uploaded CSR (verdict r1 #8: they were built on the host
// for every context and partition, 5x the solve time end to end).
//
//  * the CSC twin the reference keeps beside the CSR (matrix.py:47-57):
//    a stable radix sort of the entries by column (CUB), so rows stay
//    ascending inside every column, exactly the host counting sort's order;
//  * the per-partition segment lists of the sparse kernel (rebk_csr.cu):
//    for every block of the minor axis, the major lines with entries in it
//    (ascending), each line's [lo, hi) range, a compact copy of those
//    entries with block-relative minor indices, and each CTA's first
//    segment.  A line's entries in one block are contiguous (minor indices
//    are sorted), so a segment starts wherever the block of the minor index
//    changes along a line; segment starts are selected, stably sorted by
//    block (line order kept), and measured / copied in parallel.  The lists
//    are identical to the sequential host construction.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "rebk_internal.h"

namespace rebk {

namespace {

constexpr int kTB = 256;

inline unsigned nblocks(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + kTB - 1) / kTB); }

__global__ void k_line_of(int64_t nmajor, const int64_t* __restrict__ mptr, int32_t* __restrict__ line) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= nmajor) return;
  for (int64_t e = mptr[i] + (threadIdx.x & 31); e < mptr[i + 1]; e += 32) line[e] = (int32_t)i;
}

__global__ void k_count_cols(int64_t nnz, const int32_t* __restrict__ col, unsigned long long* __restrict__ cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) atomicAdd(cnt + col[e], 1ull);
}

__global__ void k_iota(int64_t n, int64_t* __restrict__ v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void k_gather_csc(int64_t nnz, const int64_t* __restrict__ perm, const int32_t* __restrict__ line,
                             const double* __restrict__ val, int32_t* __restrict__ row_out,
                             double* __restrict__ val_out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  const int64_t e = perm[q];
  row_out[q] = line[e];
  val_out[q] = val[e];
}

__global__ void k_ull_to_ptr(int64_t n, const unsigned long long* __restrict__ cnt, int64_t* __restrict__ ptr) {
  // ptr[0] = 0, ptr[j + 1] = inclusive sum (written by the scan); here: copy counts to int64
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) ptr[j] = (int64_t)cnt[j];
}

__global__ void k_block_of(int64_t nminor, int64_t nb, const int64_t* __restrict__ bptr, int32_t* __restrict__ blk) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nminor) return;
  int64_t lo = 0, hi = nb;  // largest q with bptr[q] <= j
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (bptr[mid] <= j) lo = mid;
    else hi = mid;
  }
  blk[j] = (int32_t)lo;
}

__global__ void k_seg_flags(int64_t nnz, const int64_t* __restrict__ mptr, const int32_t* __restrict__ line,
                            const int32_t* __restrict__ minor, const int32_t* __restrict__ blk,
                            uint8_t* __restrict__ flag) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  flag[e] = (e == mptr[line[e]] || blk[minor[e]] != blk[minor[e - 1]]) ? 1 : 0;
}

__global__ void k_seg_keys(int64_t nseg, int64_t nnz, const int64_t* __restrict__ start,
                           const int64_t* __restrict__ mptr, const int32_t* __restrict__ line,
                           const int32_t* __restrict__ minor, const int32_t* __restrict__ blk,
                           int32_t* __restrict__ key, int64_t* __restrict__ end) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int64_t e = start[s];
  const int32_t i = line[e];
  key[s] = blk[minor[e]];
  end[s] = (s + 1 < nseg && line[start[s + 1]] == i) ? start[s + 1] : mptr[i + 1];
}

__global__ void k_seg_fields(int64_t nseg, const int64_t* __restrict__ order, const int64_t* __restrict__ start,
                             const int64_t* __restrict__ end, const int32_t* __restrict__ line,
                             int32_t* __restrict__ major_id, int64_t* __restrict__ len) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nseg) return;
  const int64_t s = order[k];
  major_id[k] = line[start[s]];
  len[k] = end[s] - start[s];
}

__global__ void k_block_offsets(int64_t nb, int64_t nseg, const int32_t* __restrict__ skey, int64_t* __restrict__ off) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q > nb) return;
  int64_t lo = 0, hi = nseg;  // first k with skey[k] >= q
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (skey[mid] < q) lo = mid + 1;
    else hi = mid;
  }
  off[q] = lo;
}

__global__ void k_seg_copy(int64_t nseg, const int64_t* __restrict__ order, const int64_t* __restrict__ start,
                           const int64_t* __restrict__ ptr, const int32_t* __restrict__ skey,
                           const int64_t* __restrict__ bptr, const int32_t* __restrict__ minor,
                           const double* __restrict__ vals, double* __restrict__ val_out,
                           int32_t* __restrict__ minor_out) {
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (k >= nseg) return;
  const int64_t lo = start[order[k]], o = ptr[k], len = ptr[k + 1] - ptr[k];
  const int32_t base = (int32_t)bptr[skey[k]];
  for (int64_t t = threadIdx.x & 31; t < len; t += 32) {
    val_out[o + t] = vals[lo + t];
    minor_out[o + t] = minor[lo + t] - base;
  }
}

__global__ void k_cta_first(int64_t nb, int G, int64_t nmajor, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ major_id, int64_t* __restrict__ cta) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nb * (G + 1)) return;
  const int64_t q = idx / (G + 1);
  const int g = (int)(idx % (G + 1));
  const int32_t r0 = split_rows(nmajor, G, g);
  int64_t lo = off[q], hi = off[q + 1];  // first segment of block q with major_id >= r0
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (major_id[mid] < r0) lo = mid + 1;
    else hi = mid;
  }
  cta[idx] = lo;
}

// scratch owned for the duration of one build (freed on the stream)
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <class T>
  cudaError_t get(T** p, size_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(n, 1) * sizeof(T), st);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = (T*)q;
    return e;
  }
};

#define B_TRY(x)                       \
  do {                                 \
    cudaError_t _e = (x);              \
    if (_e != cudaSuccess) return _e;  \
  } while (0)

int bits_for(int64_t v) {
  int b = 1;
  while (b < 62 && ((int64_t)1 << b) <= v) ++b;
  return b;
}

}  // namespace

cudaError_t csr_to_csc_device(int64_t m, int64_t n, int64_t nnz, const int64_t* csr_ptr, const int32_t* csr_col,
                              const double* csr_val, int64_t* csc_ptr, int32_t* csc_row, double* csc_val,
                              cudaStream_t st) {
  Scratch S(st);
  unsigned long long* cnt;
  int32_t *line, *kout;
  int64_t *idx, *perm;
  B_TRY(S.get(&cnt, n));
  B_TRY(S.get(&line, nnz));
  B_TRY(S.get(&kout, nnz));
  B_TRY(S.get(&idx, nnz));
  B_TRY(S.get(&perm, nnz));
  B_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * n, st));
  B_TRY(cudaMemsetAsync(csc_ptr, 0, sizeof(int64_t), st));
  if (nnz > 0) {
    k_line_of<<<(unsigned)((m + kTB / 32 - 1) / (kTB / 32)), kTB, 0, st>>>(m, csr_ptr, line);
    k_count_cols<<<nblocks(nnz), kTB, 0, st>>>(nnz, csr_col, cnt);
    k_iota<<<nblocks(nnz), kTB, 0, st>>>(nnz, idx);
    B_TRY(cudaGetLastError());
  }
  k_ull_to_ptr<<<nblocks(n), kTB, 0, st>>>(n, cnt, csc_ptr + 1);
  B_TRY(cudaGetLastError());
  size_t tb = 0;
  B_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, csc_ptr + 1, csc_ptr + 1, (int)n, st));
  void* tmp;
  B_TRY(S.get((char**)&tmp, tb));
  B_TRY(cub::DeviceScan::InclusiveSum(tmp, tb, csc_ptr + 1, csc_ptr + 1, (int)n, st));
  if (nnz == 0) return cudaSuccess;
  // stable sort of entry positions by column: rows stay ascending per column
  size_t tb2 = 0;
  B_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb2, csr_col, kout, idx, perm, nnz, 0, bits_for(n), st));
  void* tmp2;
  B_TRY(S.get((char**)&tmp2, tb2));
  B_TRY(cub::DeviceRadixSort::SortPairs(tmp2, tb2, csr_col, kout, idx, perm, nnz, 0, bits_for(n), st));
  k_gather_csc<<<nblocks(nnz), kTB, 0, st>>>(nnz, perm, line, csr_val, csc_row, csc_val);
  B_TRY(cudaGetLastError());
  return cudaStreamSynchronize(st);
}

cudaError_t seg_lists_device(int64_t nmajor, const int64_t* mptr, const int32_t* minor, const double* vals,
                             int64_t nnz, int64_t nminor, int64_t nb, const int64_t* bptr_host, int G, DevSegLists* out,
                             cudaStream_t st) {
  *out = DevSegLists{};
  Scratch S(st);
  int64_t* bptr;
  int32_t *blk, *line, *key, *skey;
  uint8_t* flag;
  int64_t *start, *end, *order, *sidx, *nsel;
  B_TRY(S.get(&bptr, nb + 1));
  B_TRY(cudaMemcpyAsync(bptr, bptr_host, sizeof(int64_t) * (nb + 1), cudaMemcpyHostToDevice, st));
  B_TRY(S.get(&blk, nminor));
  B_TRY(S.get(&line, nnz));
  B_TRY(S.get(&flag, nnz));
  B_TRY(S.get(&start, nnz));
  B_TRY(S.get(&nsel, 1));
  k_block_of<<<nblocks(nminor), kTB, 0, st>>>(nminor, nb, bptr, blk);
  if (nnz > 0) {
    k_line_of<<<(unsigned)((nmajor + kTB / 32 - 1) / (kTB / 32)), kTB, 0, st>>>(nmajor, mptr, line);
    k_seg_flags<<<nblocks(nnz), kTB, 0, st>>>(nnz, mptr, line, minor, blk, flag);
  }
  B_TRY(cudaGetLastError());
  // segment starts, in entry (= line-major) order
  size_t tb = 0;
  cub::CountingInputIterator<int64_t> it(0);
  B_TRY(cub::DeviceSelect::Flagged(nullptr, tb, it, flag, start, nsel, nnz, st));
  void* tmp;
  B_TRY(S.get((char**)&tmp, tb));
  B_TRY(cub::DeviceSelect::Flagged(tmp, tb, it, flag, start, nsel, nnz, st));
  int64_t nseg = 0;
  B_TRY(cudaMemcpyAsync(&nseg, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  B_TRY(cudaStreamSynchronize(st));
  out->nseg = nseg;
  B_TRY(S.get(&key, nseg));
  B_TRY(S.get(&skey, nseg));
  B_TRY(S.get(&end, nseg));
  B_TRY(S.get(&sidx, nseg));
  B_TRY(S.get(&order, nseg));
  if (nseg > 0) {
    k_seg_keys<<<nblocks(nseg), kTB, 0, st>>>(nseg, nnz, start, mptr, line, minor, blk, key, end);
    k_iota<<<nblocks(nseg), kTB, 0, st>>>(nseg, sidx);
    B_TRY(cudaGetLastError());
    size_t tb2 = 0;
    B_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb2, key, skey, sidx, order, nseg, 0, bits_for(nb), st));
    void* tmp2;
    B_TRY(S.get((char**)&tmp2, tb2));
    B_TRY(cub::DeviceRadixSort::SortPairs(tmp2, tb2, key, skey, sidx, order, nseg, 0, bits_for(nb), st));
  }
  // outputs (owned by the plan; cudaFree in free_seg_plan)
  B_TRY(pool_malloc(&out->off, nb + 1));
  B_TRY(pool_malloc(&out->major_id, nseg));
  B_TRY(pool_malloc(&out->ptr, nseg + 1));
  B_TRY(pool_malloc(&out->cta, nb * (G + 1)));
  int64_t* len;
  B_TRY(S.get(&len, nseg));
  if (nseg > 0) {
    k_seg_fields<<<nblocks(nseg), kTB, 0, st>>>(nseg, order, start, end, line, out->major_id, len);
    B_TRY(cudaGetLastError());
  }
  k_block_offsets<<<nblocks(nb + 1), kTB, 0, st>>>(nb, nseg, skey, out->off);
  B_TRY(cudaGetLastError());
  B_TRY(cudaMemsetAsync(out->ptr, 0, sizeof(int64_t), st));
  if (nseg > 0) {
    size_t tb3 = 0;
    B_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb3, len, out->ptr + 1, (int)nseg, st));
    void* tmp3;
    B_TRY(S.get((char**)&tmp3, tb3));
    B_TRY(cub::DeviceScan::InclusiveSum(tmp3, tb3, len, out->ptr + 1, (int)nseg, st));
  }
  int64_t nent = 0;
  B_TRY(cudaMemcpyAsync(&nent, out->ptr + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  B_TRY(cudaStreamSynchronize(st));
  B_TRY(pool_malloc(&out->val, nent));
  B_TRY(pool_malloc(&out->minor_local, nent));
  if (nseg > 0) {
    k_seg_copy<<<(unsigned)((nseg + kTB / 32 - 1) / (kTB / 32)), kTB, 0, st>>>(
        nseg, order, start, out->ptr, skey, bptr, minor, vals, out->val, out->minor_local);
    B_TRY(cudaGetLastError());
  }
  k_cta_first<<<nblocks(nb * (G + 1)), kTB, 0, st>>>(nb, G, nmajor, out->off, out->major_id, out->cta);
  B_TRY(cudaGetLastError());
  return cudaStreamSynchronize(st);
}

}  // namespace rebk

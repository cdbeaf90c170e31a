// rebk_nccl.cu — the row-sharded multi-GPU iteration (BASELINE config 3,
// SURVEY §8e) driven from C++: one call runs a whole solve on this rank,
// issuing the per-rank kernels (rebk_shard.cu) and the two NCCL allreduces of
// every iteration on one stream with no host round trip per iteration.
//
// NCCL is loaded at run time (dlopen) from the path the caller passes — the
// same libnccl.so.2 torch uses — so librebk.so has no link-time NCCL
// dependency.  Per iteration (step_rebk, solvers.py:324-337):
//   u = A_p[:, J]ᵀ z_p ; allreduce(u) ; z_p -= s_J A_p[:, J] u
//   dx = A_p[I_p, :]ᵀ (A_p[I_p, :] x - b_p + z_p) ; allreduce(dx) ; x -= s_I dx
// The stop check (solvers.py:444-474) writes ||x - x*||² on the device; the
// host reads a chunk of errors at once, and when a check inside the chunk
// crosses tol the chunk is replayed from its start snapshot to exactly that
// iteration (kernels and fixed-size allreduces are deterministic).
#include <stdarg.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/rebk.h"
#include "rebk_internal.h"

namespace rebk {
namespace nccl {

// the subset of the NCCL ABI used here (nccl.h: ncclUniqueId is 128 bytes,
// ncclFloat64 = 8, ncclSum = 0)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
typedef ncclResult_t (*GetUniqueIdFn)(ncclUniqueId*);
typedef ncclResult_t (*CommInitRankFn)(ncclComm_t*, int, ncclUniqueId, int);
typedef ncclResult_t (*CommDestroyFn)(ncclComm_t);
typedef ncclResult_t (*AllReduceFn)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef const char* (*ErrStrFn)(ncclResult_t);

struct Api {
  void* handle = nullptr;
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  AllReduceFn all_reduce = nullptr;
  ErrStrFn err_str = nullptr;
};

static Api g_api;

static bool load(const char* path, char* err, size_t errlen) {
  if (g_api.handle) return true;
  void* h = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    snprintf(err, errlen, "dlopen(%s) failed: %s", path ? path : "libnccl.so.2", dlerror());
    return false;
  }
  Api a;
  a.handle = h;
  a.get_unique_id = (GetUniqueIdFn)dlsym(h, "ncclGetUniqueId");
  a.comm_init_rank = (CommInitRankFn)dlsym(h, "ncclCommInitRank");
  a.comm_destroy = (CommDestroyFn)dlsym(h, "ncclCommDestroy");
  a.all_reduce = (AllReduceFn)dlsym(h, "ncclAllReduce");
  a.err_str = (ErrStrFn)dlsym(h, "ncclGetErrorString");
  if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce || !a.err_str) {
    snprintf(err, errlen, "%s does not export the NCCL symbols librebk needs", path);
    return false;
  }
  g_api = a;
  return true;
}

struct Comm {
  ncclComm_t comm;
  int nranks, rank, device;
};

constexpr int kFloat64 = 8, kSum = 0;

}  // namespace nccl
}  // namespace rebk

using namespace rebk;

namespace {
thread_local char g_nccl_err[512];
int nfail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_nccl_err, sizeof g_nccl_err, fmt, ap);
  va_end(ap);
  return set_error_msg(code, g_nccl_err);
}
}  // namespace

extern "C" int rebk_nccl_get_unique_id(const char* libnccl_path, unsigned char id_out[128]) {
  char err[400];
  if (!id_out) return nfail(REBK_EINVAL, "rebk_nccl_get_unique_id: null output");
  if (!nccl::load(libnccl_path, err, sizeof err)) return nfail(REBK_EINVAL, "%s", err);
  nccl::ncclUniqueId id;
  const int r = nccl::g_api.get_unique_id(&id);
  if (r != 0) return nfail(REBK_ECUDA, nccl::g_api.err_str(r));
  memcpy(id_out, id.internal, 128);
  return REBK_OK;
}

extern "C" int rebk_nccl_comm_create(const char* libnccl_path, const unsigned char id[128], int nranks, int rank,
                                     int device, void** comm_out) {
  char err[400];
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return nfail(REBK_EINVAL, "rebk_nccl_comm_create: bad argument");
  if (!nccl::load(libnccl_path, err, sizeof err)) return nfail(REBK_EINVAL, "%s", err);
  if (cudaSetDevice(device) != cudaSuccess) return nfail(REBK_ENODEV, "rebk_nccl_comm_create: no such device");
  nccl::ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  nccl::ncclComm_t c = nullptr;
  const int r = nccl::g_api.comm_init_rank(&c, nranks, uid, rank);
  if (r != 0) return nfail(REBK_ECUDA, nccl::g_api.err_str(r));
  *comm_out = new nccl::Comm{c, nranks, rank, device};
  return REBK_OK;
}

extern "C" int rebk_nccl_comm_destroy(void* comm) {
  if (!comm) return REBK_OK;
  nccl::Comm* c = (nccl::Comm*)comm;
  if (nccl::g_api.comm_destroy) nccl::g_api.comm_destroy(c->comm);
  delete c;
  return REBK_OK;
}

extern "C" int rebk_shard_run(rebk_ctx* ctx, void* comm, const rebk_shard_run_args* a, int64_t* iters_out,
                              int32_t* converged_out, double* final_err_out) {
  if (!ctx || !comm || !a || !a->picks || !a->row_ptr || !a->row_scale || !a->local_ranges || !a->local_rows_dev ||
      !a->b_dev || !a->x_dev || !a->xs_dev || a->max_iters < 0 || a->stride < 1 || a->chunk < 1 ||
      (a->extended && (!a->col_ptr || !a->col_scale || !a->z_dev)))
    return nfail(REBK_EINVAL, "rebk_shard_run: bad argument");
  if (a->n_picks < a->max_iters) return nfail(REBK_EINVAL, "rebk_shard_run: %lld picks for %lld iterations",
                                              (long long)a->n_picks, (long long)a->max_iters);
  for (int64_t k = 0; k < a->max_iters; ++k) {
    const int32_t jb = a->picks[2 * k], ib = a->picks[2 * k + 1];
    if (ib < 0 || ib >= a->n_row_blocks || (a->extended && (jb < 0 || jb >= a->n_col_blocks)))
      return nfail(REBK_EINVAL, "rebk_shard_run: pick %lld = (%d, %d) out of range", (long long)k, jb, ib);
  }
  nccl::Comm* cm = (nccl::Comm*)comm;
  const double* A = nullptr;
  int64_t m = 0, n = 0, lda = 0;
  int ctx_dev = 0;
  if (!ctx_dense_view(ctx, &A, &m, &n, &lda, &ctx_dev) || !A)
    return nfail(REBK_EINVAL, "rebk_shard_run: dense context required");
  if (cudaSetDevice(cm->device) != cudaSuccess) return nfail(REBK_ENODEV, "rebk_shard_run: no device");
  int64_t nJmax = 1, nImax = 1;
  if (a->extended)
    for (int64_t j = 0; j < a->n_col_blocks; ++j) nJmax = std::max(nJmax, a->col_ptr[j + 1] - a->col_ptr[j]);
  for (int64_t i = 0; i < a->n_row_blocks; ++i)
    nImax = std::max(nImax, a->local_ranges[2 * i + 1] - a->local_ranges[2 * i]);
  if (nJmax > 512) return nfail(REBK_EINVAL, "rebk_shard_run: column blocks up to 512 wide");

  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nfail(REBK_ECUDA, "stream");
  const int chunk = a->chunk;
  double *u = nullptr, *dx = nullptr, *scr_c = nullptr, *scr_r = nullptr, *errs = nullptr, *x0 = nullptr,
         *z0 = nullptr;
  cudaError_t e = cudaSuccess;
  auto alloc = [&](double** p, size_t cnt) {
    if (e == cudaSuccess) e = cudaMallocAsync((void**)p, std::max<size_t>(cnt, 1) * sizeof(double), st);
  };
  alloc(&u, nJmax);
  alloc(&dx, n);
  alloc(&scr_c, a->extended ? shard_colstep_scratch(std::max<int64_t>(m, 1), nJmax) : 1);
  alloc(&scr_r, shard_rowstep_scratch(nImax, n));
  alloc(&errs, chunk);
  alloc(&x0, n);
  alloc(&z0, std::max<int64_t>(m, 1));
  std::vector<double> herr(chunk);
  int rc = REBK_OK;
  const bool have_rows = m > 0;
  // every rank agrees that setup succeeded before anyone enters a collective
  // of the iteration loop (a rank that failed alone would leave its peers
  // blocked in ncclAllReduce): allreduce one failure flag
  {
    double* flag = nullptr;
    const double mine = e == cudaSuccess ? 0.0 : 1.0;
    double any = 1.0;
    cudaGetLastError();
    cudaError_t fe = cudaMallocAsync((void**)&flag, sizeof(double), st);
    if (fe == cudaSuccess) fe = cudaMemcpyAsync(flag, &mine, sizeof(double), cudaMemcpyHostToDevice, st);
    if (fe == cudaSuccess &&
        nccl::g_api.all_reduce(flag, flag, 1, nccl::kFloat64, nccl::kSum, cm->comm, st) != 0)
      fe = cudaErrorUnknown;
    if (fe == cudaSuccess) fe = cudaMemcpyAsync(&any, flag, sizeof(double), cudaMemcpyDeviceToHost, st);
    if (fe == cudaSuccess) fe = cudaStreamSynchronize(st);
    if (flag) cudaFreeAsync(flag, st);
    if (e == cudaSuccess && (fe != cudaSuccess || any != 0.0)) e = fe != cudaSuccess ? fe : cudaErrorMemoryAllocation;
  }

  auto iterate = [&](int64_t k) -> cudaError_t {
    const int jb = a->picks[2 * (k - 1)], ib = a->picks[2 * (k - 1) + 1];
    cudaError_t ce = cudaSuccess;
    if (a->extended) {
      const int64_t c_lo = a->col_ptr[jb], nJ = a->col_ptr[jb + 1] - c_lo;
      if (have_rows) ce = shard_colstep(A, lda, m, c_lo, (int)nJ, a->z_dev, u, scr_c, st);
      else ce = cudaMemsetAsync(u, 0, nJ * sizeof(double), st);
      if (ce != cudaSuccess) return ce;
      if (nccl::g_api.all_reduce(u, u, (size_t)nJ, nccl::kFloat64, nccl::kSum, cm->comm, st) != 0)
        return cudaErrorUnknown;
      if (have_rows) ce = shard_zupd(A, lda, m, c_lo, (int)nJ, a->col_scale[jb], u, a->z_dev, st);
      if (ce != cudaSuccess) return ce;
    }
    const int64_t lo = a->local_ranges[2 * ib], hi = a->local_ranges[2 * ib + 1];
    ce = shard_rowstep(A, lda, n, a->local_rows_dev + lo, hi - lo, a->x_dev, a->b_dev,
                       a->extended ? a->z_dev : nullptr, scr_r, dx, st);
    if (ce != cudaSuccess) return ce;
    if (nccl::g_api.all_reduce(dx, dx, (size_t)n, nccl::kFloat64, nccl::kSum, cm->comm, st) != 0)
      return cudaErrorUnknown;
    return shard_xupd(n, a->row_scale[ib], dx, a->x_dev, st);
  };

  int64_t iters = 0;
  int32_t converged = 0;
  double final_err = NAN;
  // check at k = 0
  if (e == cudaSuccess) e = shard_err(n, a->x_dev, a->xs_dev, errs, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(herr.data(), errs, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    final_err = sqrt(herr[0]);
    converged = final_err <= a->tol;
  }
  int64_t k = 0;
  while (e == cudaSuccess && !converged && k < a->max_iters) {
    const int64_t cnt = std::min<int64_t>(chunk, a->max_iters - k);
    e = cudaMemcpyAsync(x0, a->x_dev, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && a->extended && have_rows)
      e = cudaMemcpyAsync(z0, a->z_dev, m * sizeof(double), cudaMemcpyDeviceToDevice, st);
    int64_t last_check = -1;
    for (int64_t t = 0; t < cnt && e == cudaSuccess; ++t) {
      e = iterate(k + t + 1);
      if (e == cudaSuccess && (k + t + 1) % a->stride == 0) {
        e = shard_err(n, a->x_dev, a->xs_dev, errs + t, st);
        last_check = t;
      }
    }
    if (e == cudaSuccess && last_check >= 0) {
      e = cudaMemcpyAsync(herr.data(), errs, cnt * sizeof(double), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      int64_t hit = -1;
      for (int64_t t = 0; e == cudaSuccess && t < cnt; ++t)
        if ((k + t + 1) % a->stride == 0 && sqrt(herr[t]) <= a->tol) {
          hit = t;
          break;
        }
      if (hit >= 0) {
        if (hit + 1 < cnt) {  // replay the chunk to exactly the crossing iteration
          e = cudaMemcpyAsync(a->x_dev, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
          if (e == cudaSuccess && a->extended && have_rows)
            e = cudaMemcpyAsync(a->z_dev, z0, m * sizeof(double), cudaMemcpyDeviceToDevice, st);
          for (int64_t t = 0; t <= hit && e == cudaSuccess; ++t) e = iterate(k + t + 1);
        }
        converged = 1;
        iters = k + hit + 1;
        final_err = sqrt(herr[hit]);
        break;
      }
      final_err = sqrt(herr[last_check]);
    }
    k += cnt;
  }
  if (e == cudaSuccess && !converged) {
    iters = a->max_iters;
    if (a->max_iters % a->stride != 0) {
      e = shard_err(n, a->x_dev, a->xs_dev, errs, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(herr.data(), errs, sizeof(double), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) {
        final_err = sqrt(herr[0]);
        converged = final_err <= a->tol;
      }
    }
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    snprintf(g_nccl_err, sizeof g_nccl_err, "rebk_shard_run failed: %s", cudaGetErrorString(e));
    rc = set_error_msg(REBK_ECUDA, g_nccl_err);
  }
  for (double* p : {u, dx, scr_c, scr_r, errs, x0, z0})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc == REBK_OK) {
    if (iters_out) *iters_out = iters;
    if (converged_out) *converged_out = converged;
    if (final_err_out) *final_err_out = final_err;
  }
  return rc;
}

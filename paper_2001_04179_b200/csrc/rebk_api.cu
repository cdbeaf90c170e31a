// rebk_api.cu — the extern "C" boundary of librebk.so (declared in include/rebk.h).
//
// Host orchestration of one run (solvers.py:425-474): validate, upload the
// per-run vectors, expand the block-index stream into per-iteration plans on
// the device, launch the persistent kernel over chunks of iterations, read
// back the iterates and the RunTrace fields.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include <mutex>

#include "../../include/rebk.h"
#include "philox.h"
#include "rebk_internal.h"

using namespace rebk;

// Per-partition segment lists of the sparse kernel (built once, cached).
struct CsrSegPlan {
  std::vector<int64_t> row_ptr, col_ptr;  // the partition (cache key) and the grid size
  int G = 0;
  int64_t *cseg_off = nullptr, *cseg_ptr = nullptr, *cseg_cta = nullptr;
  int32_t *cseg_row = nullptr, *ccol = nullptr;
  double* cval = nullptr;
  int64_t *rseg_off = nullptr, *rseg_ptr = nullptr, *rseg_cta = nullptr;
  int32_t *rseg_col = nullptr, *rrow = nullptr;
  double* rval = nullptr;
};

struct rebk_ctx {
  int device;
  int kind;  // 0 dense, 1 CSR
  int64_t m, n, lda;
  const double* A;    // device (dense)
  double* A_owned;    // non-null when the ctx allocated A
  int sm_count;
  // CSR + CSC twin (device) and host copies for building segment lists
  int64_t nnz = 0;
  int64_t *csr_ptr = nullptr, *csc_ptr = nullptr;
  int32_t *csr_col = nullptr, *csc_row = nullptr;
  double *csr_val = nullptr, *csc_val = nullptr;
  std::vector<CsrSegPlan*> seg_cache;  // guarded by mu
  float* A32 = nullptr;  // dense fp32 A (multi-RHS contexts, kind 2)
  float* A32t = nullptr;  // its transpose (n x ldat), built at the first tensor-core run (under mu)
  std::mutex mu;  // lazily built caches: seg_cache, A32t (concurrent runs on one ctx)
  int64_t ldat = 0;
  double* shard_scratch = nullptr;  // rebk_shard_* partials (not reentrant per ctx)
  size_t shard_scratch_len = 0;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(_e == cudaErrorMemoryAllocation ? REBK_ENOMEM : REBK_ECUDA, "%s: %s", #expr, \
                  cudaGetErrorString(_e));                                                 \
  } while (0)

// RAII bundle of per-run device allocations, freed on the run's stream.
struct DevArena {
  cudaStream_t stream = nullptr;
  std::vector<void*> ptrs;
  ~DevArena() {
    for (void* p : ptrs) cudaFreeAsync(p, stream);
  }
  template <typename T>
  cudaError_t alloc(T** out, size_t count) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), stream);
    if (e == cudaSuccess) ptrs.push_back(p);
    *out = (T*)p;
    return e;
  }
};

int check_partition(const char* what, int64_t nb, const int64_t* ptr, const double* cum,
                    const double* scale, int64_t axis_len) {
  if (nb < 1 || !ptr || !cum || !scale)
    return fail(REBK_EINVAL, "%s partition: need at least one block with ptr/cum/scale arrays", what);
  if (ptr[0] != 0 || ptr[nb] != axis_len)
    return fail(REBK_EINVAL, "%s partition covers [%lld, %lld), matrix axis has %lld", what,
                (long long)ptr[0], (long long)ptr[nb], (long long)axis_len);
  for (int64_t b = 0; b < nb; ++b)
    if (ptr[b + 1] <= ptr[b]) return fail(REBK_EINVAL, "empty block in %s partition", what);
  return REBK_OK;
}

int max_block(int64_t nb, const int64_t* ptr) {
  int64_t mx = 0;
  for (int64_t b = 0; b < nb; ++b) mx = std::max(mx, ptr[b + 1] - ptr[b]);
  return (int)mx;
}

int env_int(const char* name, int dflt);

bool blocks_even(int64_t nb, const int64_t* ptr) {
  for (int64_t b = 0; b < nb; ++b)
    if (ptr[b] & 1) return false;
  return true;
}

int grid_override() {
  const char* s = getenv("REBK_GRID");
  return s ? atoi(s) : 0;
}

// The persistent kernel's grid size depends only on the matrix shape, so two
// runs on one matrix (e.g. rebk with z0 = 0 and rabk) do bit-identical row
// sweeps (test_solvers.py:249-265).
int choose_grid(const rebk_ctx* ctx, const rebk_cfg* cfg, int max_resident) {
  int G = cfg->grid_ctas > 0 ? cfg->grid_ctas : grid_override();
  if (G <= 0) {
    const int64_t cells = ctx->m * ctx->n;
    G = (int)std::min<int64_t>((cells + 65535) / 65536, (int64_t)ctx->sm_count);
  }
  G = std::max(1, std::min(G, max_resident));
  return G;
}

struct Geometry {
  int G;
  int nR_max, nC_max, nJ_max, nI_max;
  int ct_ld, rt_ld;
  int stage_ct, stage_rt;
  int ct_off, rt_off, vec_off;
  size_t smem_bytes;
};

Geometry plan_geometry(const rebk_ctx* ctx, const rebk_cfg* cfg, int G, bool extended) {
  Geometry g{};
  g.G = G;
  for (int q = 0; q < G; ++q) {
    g.nR_max = std::max(g.nR_max, split_rows(ctx->m, G, q + 1) - split_rows(ctx->m, G, q));
    g.nC_max = std::max(g.nC_max, split_even(ctx->n, G, q + 1) - split_even(ctx->n, G, q));
  }
  g.nI_max = max_block(cfg->n_row_blocks, cfg->row_ptr);
  g.nJ_max = extended ? max_block(cfg->n_col_blocks, cfg->col_ptr) : 0;
  g.ct_ld = (g.nJ_max + 1) & ~1;
  g.rt_ld = ((g.nC_max + 1) & ~1);
  if (g.rt_ld % 4 == 0) g.rt_ld += 2;  // ≡ 2 (mod 4): conflict-free 2-lane row reads
  const size_t vec = (size_t)(2 * g.nC_max + g.nR_max + g.nJ_max + g.nI_max + kThreads);
  const size_t ct = (size_t)g.nR_max * g.ct_ld;
  const size_t rt = (size_t)g.nI_max * g.rt_ld;
  const size_t budget = (size_t)kSmemBudget / 8;
  const bool aligned = (ctx->lda % 2 == 0) && ((uintptr_t)ctx->A % 16 == 0);
  const bool ct_ok = aligned && extended && g.nJ_max >= 2 &&
                     blocks_even(cfg->n_col_blocks, cfg->col_ptr);
  const bool rt_ok = aligned && g.nC_max >= 2;
  const char* no_stage = getenv("REBK_NO_STAGE");
  const bool allow = !(no_stage && no_stage[0] == '1');
  g.stage_ct = g.stage_rt = 0;
  if (allow && ct_ok && rt_ok && vec + ct + rt <= budget) {
    g.stage_ct = g.stage_rt = 1;
  } else if (allow && rt_ok && vec + rt <= budget) {
    g.stage_rt = 1;
  } else if (allow && ct_ok && vec + ct <= budget) {
    g.stage_ct = 1;
  }
  size_t off = 0;
  g.ct_off = (int)off;
  if (g.stage_ct) off += ct;
  g.rt_off = (int)off;
  if (g.stage_rt) off += rt;
  g.vec_off = (int)off;
  off += vec;
  g.smem_bytes = off * 8;
  return g;
}

// The general kernel falls back to unstaged (global-memory) tile reads when a
// tile is not TMA-able (odd column-block starts, 1-wide blocks) and when it is
// too large for shared memory.  Only the second case goes to the streaming
// kernel: small unaligned problems keep the general kernel's summation order,
// so e.g. REBK with z0 = 0 stays bitwise equal to RABK (test_solvers.py:249-265).
bool tiles_exceed_smem(const Geometry& g, bool extended) {
  const size_t vec = (size_t)(2 * g.nC_max + g.nR_max + g.nJ_max + g.nI_max + kThreads);
  const size_t budget = (size_t)kSmemBudget / 8;
  if (vec + (size_t)g.nI_max * g.rt_ld > budget) return true;
  return extended && vec + (size_t)g.nR_max * g.ct_ld > budget;
}

// ---- fast path (rebk_dense_fast.cu) -------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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

bool encode_box(CUtensorMap* map, const rebk_ctx* ctx, int box_w, int box_h) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)ctx->n, (cuuint64_t)ctx->m};
  cuuint64_t gstride[1] = {(cuuint64_t)ctx->lda * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)ctx->A, gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int round_even(int v) { return (v + 1) & ~1; }

struct FastGeometry {
  bool ok = false;
  int G = 0, CS = 0, NC = 0;
  int nR_max = 0, nC_max = 0, nJ_max = 0, nI_max = 0;
  int ct_box_w = 0, ct_box_h = 0, rt_box_w = 0, rt_box_h = 0;
  int pad_nC = 0, pad_nR = 0, pad_ne = 0, pad_in = 0, pad_cin = 0;
  int ct_off = 0, rt_off = 0, vec_off = 0;
  int vec_off_c = 0, vec_off_r = 0;  // split path: per-group vector bases
  int pieces = 1;                    // split path: TMA boxes per tile
  size_t smem_bytes = 0;
};

FastGeometry fast_geometry(const rebk_ctx* ctx, const rebk_cfg* cfg, bool extended, int NC, int CS) {
  FastGeometry f;
  f.CS = CS;
  f.NC = NC;
  f.G = NC * CS;
  const int G = f.G;
  for (int q = 0; q < G; ++q) {
    f.nR_max = std::max(f.nR_max, split_rows(ctx->m, G, q + 1) - split_rows(ctx->m, G, q));
    f.nC_max = std::max(f.nC_max, split_even(ctx->n, G, q + 1) - split_even(ctx->n, G, q));
  }
  f.nI_max = max_block(cfg->n_row_blocks, cfg->row_ptr);
  f.nJ_max = extended ? max_block(cfg->n_col_blocks, cfg->col_ptr) : 0;
  f.ct_box_w = extended ? std::max(2, round_even(f.nJ_max)) : 2;
  f.ct_box_h = extended ? std::max(1, f.nR_max) : 1;
  f.rt_box_w = std::max(2, round_even(f.nC_max));
  if (f.rt_box_w % 4 == 0) f.rt_box_w += 2;  // ≡ 2 (mod 4) doubles: conflict-free row-parallel reads
  f.rt_box_h = f.nI_max;
  if (f.ct_box_w > 256 || f.ct_box_h > 256 || f.rt_box_w > 256 || f.rt_box_h > 256) return f;
  const int ne_max = std::max(f.nJ_max, 2 * f.nI_max) + 1;
  const int sl = (ne_max + CS - 1) / CS;
  f.pad_nC = round_even(f.nC_max + 1);
  f.pad_nR = round_even(f.nR_max + 1);
  f.pad_ne = round_even(ne_max + 1);
  f.pad_in = round_even(CS * sl);
  f.pad_cin = round_even(NC * sl);
  auto al16 = [](size_t v) { return (v + 15) & ~(size_t)15; };  // 128-byte alignment in doubles
  size_t off = 0;
  f.ct_off = (int)off;
  off = al16(off + (size_t)f.ct_box_w * f.ct_box_h);
  f.rt_off = (int)off;
  off = al16(off + (size_t)f.rt_box_w * f.rt_box_h);
  f.vec_off = (int)off;
  off += 2 * (size_t)f.pad_nC + f.pad_nR + 3 * (size_t)f.pad_ne + f.pad_in + f.pad_cin + 2 * kThreads;
  f.smem_bytes = off * sizeof(double);
  f.ok = f.smem_bytes <= (size_t)kSmemBudget;
  return f;
}

// Split path geometry: clusters [0, ncc) sweep columns (z rows split over
// ncc*CS CTAs), the rest sweep rows (x columns split over the remaining CTAs).
FastGeometry split_geometry(const rebk_ctx* ctx, const rebk_cfg* cfg, int NC, int CS, int ncc, int xmode, int pieces) {
  FastGeometry f;
  f.CS = CS;
  f.NC = NC;
  f.G = NC * CS;
  const int Gc = ncc * CS, Gr = (NC - ncc) * CS;
  for (int q = 0; q < Gc; ++q)
    f.nR_max = std::max(f.nR_max, split_rows(ctx->m, Gc, q + 1) - split_rows(ctx->m, Gc, q));
  for (int q = 0; q < Gr; ++q)
    f.nC_max = std::max(f.nC_max, split_even(ctx->n, Gr, q + 1) - split_even(ctx->n, Gr, q));
  f.nI_max = max_block(cfg->n_row_blocks, cfg->row_ptr);
  f.nJ_max = max_block(cfg->n_col_blocks, cfg->col_ptr);
  f.ct_box_w = std::max(2, round_even(f.nJ_max));
  // pieces == 2: each tile arrives as two half-height boxes (rows [0, h) and
  // [h, 2h)) on two mbarriers, so the next tile's first half loads while the
  // second half is still being consumed; pieces == 1: one box per tile
  f.pieces = pieces;
  f.ct_box_h = std::max(1, (f.nR_max + pieces - 1) / pieces);
  f.rt_box_w = std::max(2, round_even(f.nC_max));
  if (f.rt_box_w % 4 == 0) f.rt_box_w += 2;
  f.rt_box_h = std::max(1, (f.nI_max + pieces - 1) / pieces);
  if (f.ct_box_w > 256 || f.ct_box_h > 256 || f.rt_box_w > 256 || f.rt_box_h > 256) return f;
  const int ne_max = std::max(f.nJ_max, f.nI_max) + 1;
  const int sl = (ne_max + CS - 1) / CS;
  f.pad_nC = round_even(f.nC_max + 1);
  f.pad_nR = round_even(f.nR_max + 1);
  f.pad_ne = round_even(ne_max + 1);
  f.pad_in = round_even(CS * sl);
  f.pad_cin = round_even(std::max(ncc, NC - ncc) * ne_max);  // all entries from every cluster
  auto al16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
  // per-group layouts after the group's own tile:
  //   column group: [tile][z][u r part][in][red][cin over ncc clusters]
  //   row group:    [tile][x xs][u r part][in][red][cin over NC-ncc clusters]
  f.ct_off = f.rt_off = 0;
  f.vec_off_c = (int)(pieces * al16((size_t)f.ct_box_w * f.ct_box_h));
  f.vec_off_r = (int)(pieces * al16((size_t)f.rt_box_w * f.rt_box_h));
  f.vec_off = f.vec_off_c;
  const size_t common = 3 * (size_t)f.pad_ne + f.pad_in + 2 * 512;  // 2*512: colsum2<512> scratch
  // s_cin: a gather-all exchange keeps every cluster's partials of every
  // entry, a broadcast exchange only those of the CTA's slice
  const int gather_c = xmode & 1, gather_r = (xmode >> 1) & 1;
  const size_t cin_c = (size_t)ncc * (gather_c ? ne_max : sl), cin_r = (size_t)(NC - ncc) * (gather_r ? ne_max : sl);
  const size_t need_c = f.vec_off_c + (size_t)f.pad_nR + common + cin_c;
  const size_t need_r = f.vec_off_r + 2 * (size_t)f.pad_nC + common + cin_r;
  f.pad_cin = round_even((int)std::max(cin_c, cin_r));
  f.smem_bytes = std::max(need_c, need_r) * sizeof(double);
  f.ok = f.smem_bytes <= (size_t)kSmemBudget;
  return f;
}

// Streaming path geometry (rebk_dense_stream.cu): G CTAs, one per SM; the
// vectors go after a ring of NS stages that takes the rest of the budget.
struct StreamGeometry {
  bool ok = false;
  int G = 0, NS = 0, SD = 0, cw = 0, ch = 0, rw = 0, rh = 0, lc = 0, lr = 0;
  int nR_max = 0, nC_max = 0, nJ_max = 0, nI_max = 0;
  int pad_nC = 0, pad_nR = 0, pad_nJ = 0, pad_nI = 0;
  size_t smem_bytes = 0;
};

int pow2floor_host(int v) {
  int p = 1;
  while (p * 2 <= v) p *= 2;
  return p;
}

// m rows split over G CTAs, n columns split over G CTAs; the largest row /
// column block; odd column-block starts need one extra leading column
StreamGeometry stream_geometry_dims(int64_t m, int64_t n, int nI_max, int nJ_max, bool cols_even, int G,
                                    bool extended) {
  StreamGeometry f;
  f.G = G;
  for (int q = 0; q < G; ++q) {
    f.nR_max = std::max(f.nR_max, split_rows(m, G, q + 1) - split_rows(m, G, q));
    f.nC_max = std::max(f.nC_max, split_even(n, G, q + 1) - split_even(n, G, q));
  }
  f.nI_max = nI_max;
  f.nJ_max = extended ? nJ_max : 0;
  f.pad_nC = round_even(f.nC_max + 1);
  f.pad_nR = extended ? round_even(f.nR_max + 1) : 0;
  f.pad_nJ = round_even(f.nJ_max + 2);  // + a leading column for odd block starts
  f.pad_nI = round_even(f.nI_max + 1);
  const size_t vec = 2 * (size_t)f.pad_nC + f.pad_nR + f.pad_nJ + f.pad_nI + 2 * 512;
  const size_t budget = (size_t)kSmemBudget / 8;
  if (vec + 4 * 1024 > budget) return f;  // z slice too large for the on-chip vectors
  // two large stages measured best on C3 (profiles/r01_c3_stream.txt): HBM
  // runs at its copy peak on the column passes with ~95 KB boxes
  f.NS = std::max(2, std::min(kStreamMaxStages, env_int("REBK_STREAM_NS", 2)));
  f.SD = (int)(((budget - vec) / f.NS) & ~(size_t)15);
  const int hcap = std::max(1, std::min(256, env_int("REBK_STREAM_HCAP", 256)));
  // boxes: widths <= 256 elements, even; heights so a box fills a stage and
  // each row gets at least 8 lanes in the row dots (bank-conflict free)
  auto width = [](int len) {
    const int nsub = std::max(1, (len + 255) / 256);
    return std::max(2, round_even((len + nsub - 1) / nsub));
  };
  if (extended) {
    f.cw = width(f.nJ_max + (cols_even ? 0 : 1));
    f.ch = std::max(1, std::min({f.SD / f.cw, hcap, std::max(1, f.nR_max)}));
    f.lc = std::min(32, pow2floor_host(512 / f.ch));
  }
  f.rw = width(std::max(f.nC_max, 2));
  f.rh = std::max(1, std::min({f.SD / f.rw, hcap, std::max(1, f.nI_max)}));
  f.lr = std::min(32, pow2floor_host(512 / f.rh));
  f.smem_bytes = ((size_t)f.NS * f.SD + vec) * sizeof(double);
  f.ok = f.smem_bytes <= (size_t)kSmemBudget;
  return f;
}

StreamGeometry stream_geometry(const rebk_ctx* ctx, const rebk_cfg* cfg, int G, bool extended) {
  return stream_geometry_dims(ctx->m, ctx->n, max_block(cfg->n_row_blocks, cfg->row_ptr),
                              extended ? max_block(cfg->n_col_blocks, cfg->col_ptr) : 0,
                              !extended || blocks_even(cfg->n_col_blocks, cfg->col_ptr), G, extended);
}

// REBK_PROF tables: per-iteration microseconds per mark, mean and max over
// CTAs; CTAs [0, gsplit) and [gsplit, G) get separate tables (split path).
void print_prof(const std::vector<long long>& h, int G, int gsplit, int khz, double it) {
  for (int grp = 0; grp < (gsplit < G ? 2 : 1); ++grp) {
    const int q0 = grp ? gsplit : 0, q1 = grp ? G : gsplit;
    if (gsplit < G) fprintf(stderr, "[rebk prof] %s group, %d CTAs\n", grp ? "row" : "column", q1 - q0);
    double tot = 0;
    for (int i = 0; i < 16; ++i) {
      double mean = 0, mx = 0;
      for (int q = q0; q < q1; ++q) {
        const double v = (double)h[(size_t)q * 16 + i] / (khz * 1e-3) / it;
        mean += v / (q1 - q0);
        mx = std::max(mx, v);
      }
      tot += mean;
      if (mx > 0) fprintf(stderr, "[rebk prof] %2d %8.3f %8.3f\n", i, mean, mx);
    }
    fprintf(stderr, "[rebk prof] sum %8.3f\n", tot);
  }
}

int env_int(const char* name, int dflt);
// Streaming kernel, L2 retention of the column pass (StreamParams.tail): when
// the launch's slice of a column block plus its slice of a row block fit in
// L2 (a rank of a sharded run: 100 + 10 MB at C3 / 8), every C1 box is loaded
// evict_last and the C2 pass re-reads the slice from L2 (measured on that
// shape, one GPU: 44.7 -> 38.8 us per iteration); otherwise C1 streams
// evict_first (C3 on one GPU: 800 MB).  REBK_STREAM_TAIL overrides (chunks
// from the end of C1 to keep).
int stream_tail(const rebk_ctx* ctx, int64_t rows_in_launch, int nJ_max, int64_t nI_rows_in_launch, bool extended) {
  const int forced = env_int("REBK_STREAM_TAIL", -1);
  if (forced >= 0) return forced;
  if (!extended) return 0;
  int l2 = 0;
  if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device) != cudaSuccess || l2 <= 0) return 0;
  const double need = 8.0 * ((double)rows_in_launch * nJ_max + (double)nI_rows_in_launch * (double)ctx->n);
  return need <= 0.9 * (double)l2 ? (1 << 30) : 0;
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}

// ---- sparse path ---------------------------------------------------------------
bool same_vec(const std::vector<int64_t>& a, const int64_t* b, int64_t n) {
  if ((int64_t)a.size() != n) return false;
  for (int64_t i = 0; i < n; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

template <typename T>
cudaError_t upload_vec(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(dst, std::max<size_t>(v.size(), 1) * sizeof(T));
  if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

void free_seg_plan(CsrSegPlan* sp) {
  if (!sp) return;
  for (void* p : {(void*)sp->cseg_off, (void*)sp->cseg_ptr, (void*)sp->cseg_cta, (void*)sp->cseg_row, (void*)sp->ccol,
                  (void*)sp->cval, (void*)sp->rseg_off, (void*)sp->rseg_ptr, (void*)sp->rseg_cta, (void*)sp->rseg_col,
                  (void*)sp->rrow, (void*)sp->rval})
    pool_free(p);
  delete sp;
}

template <class F>
void parallel_for_threads(int T, F&& f) {
  std::vector<std::thread> pool;
  for (int th = 1; th < T; ++th) pool.emplace_back(f, th);
  f(0);
  for (auto& t : pool) t.join();
}

// Segment lists of one partition: for every column block, the rows with
// nonzeros in it and their [lo, hi) range in the CSR arrays (sorted by row);
// for every row block, the columns with nonzeros in it and their range in the
// CSC arrays (sorted by column); plus each CTA's first segment.
int build_seg_plan(rebk_ctx* ctx, const rebk_cfg* cfg, bool extended, int G, CsrSegPlan** out) {
  const int64_t s = cfg->n_row_blocks, t = extended ? cfg->n_col_blocks : 0;
  // one builder at a time; a plan is published (push_back) only after its
  // synchronous uploads completed, and plans are never freed before the ctx
  std::lock_guard<std::mutex> lock(ctx->mu);
  for (CsrSegPlan* c : ctx->seg_cache) {
    if (c->G == G && same_vec(c->row_ptr, cfg->row_ptr, s + 1) &&
        (!extended || same_vec(c->col_ptr, cfg->col_ptr, t + 1))) {
      *out = c;
      return REBK_OK;
    }
  }
  const int64_t m = ctx->m, n = ctx->n;
  CsrSegPlan* sp = new CsrSegPlan();
  sp->G = G;
  sp->row_ptr.assign(cfg->row_ptr, cfg->row_ptr + s + 1);
  if (extended) sp->col_ptr.assign(cfg->col_ptr, cfg->col_ptr + t + 1);
  // built on the device from the resident CSR / CSC (rebk_csr_build.cu)
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DevSegLists C, R;
  cudaError_t e = cudaSuccess;
  // column blocks -> row segments into CSR
  if (extended) e = seg_lists_device(m, ctx->csr_ptr, ctx->csr_col, ctx->csr_val, ctx->nnz, n, t, cfg->col_ptr, G, &C, st);
  // row blocks -> column segments into CSC
  if (!e) e = seg_lists_device(n, ctx->csc_ptr, ctx->csc_row, ctx->csc_val, ctx->nnz, m, s, cfg->row_ptr, G, &R, st);
  if (!e && !extended) {  // RABK / RK / DSBGS: an empty column plan (off = ptr = {0})
    e = pool_malloc(&C.off, 1);
    if (!e) e = pool_malloc(&C.ptr, 1);
    if (!e) e = cudaMemset(C.off, 0, sizeof(int64_t));
    if (!e) e = cudaMemset(C.ptr, 0, sizeof(int64_t));
  }
  cudaStreamDestroy(st);
  sp->cseg_off = C.off;
  sp->cseg_ptr = C.ptr;
  sp->cval = C.val;
  sp->ccol = C.minor_local;
  sp->cseg_row = C.major_id;
  sp->cseg_cta = C.cta;
  sp->rseg_off = R.off;
  sp->rseg_ptr = R.ptr;
  sp->rval = R.val;
  sp->rrow = R.minor_local;
  sp->rseg_col = R.major_id;
  sp->rseg_cta = R.cta;
  if (e) {
    free_seg_plan(sp);
    return fail(REBK_ENOMEM, "segment lists (device build) failed: %s", cudaGetErrorString(e));
  }
  ctx->seg_cache.push_back(sp);
  *out = sp;
  return REBK_OK;
}

// The sampler arrays of a run (row / column partitions, DSBGS tables,
// explicit picks) copied to the device and wired into the plan sampler.
// `cols` = the run uses the column partition (REBK/REK column sweep, or the
// DSBGS column draw).
int upload_sampler(DevArena& arena, const rebk_cfg* cfg, bool extended, bool cols, cudaStream_t stream,
                   SampleParams* sp) {
  const int64_t s = cfg->n_row_blocks, t = cols ? cfg->n_col_blocks : 0;
  const bool dsbgs = cfg->algorithm == REBK_ALGO_DSBGS;
  *sp = SampleParams{};
  sp->key0 = cfg->philox_key[0];
  sp->key1 = cfg->philox_key[1];
  sp->draw_offset = cfg->draw_offset;
  sp->extended = extended;
  sp->dsbgs = dsbgs;
  sp->n_row_blocks = (int32_t)s;
  sp->n_col_blocks = (int32_t)t;
  sp->row_total = cfg->row_total;
  sp->col_total = cfg->col_total;
  auto up = [&](auto** dst, const auto* src, int64_t count) -> cudaError_t {
    using T = std::remove_const_t<std::remove_pointer_t<decltype(src)>>;
    T* d = nullptr;
    cudaError_t e = arena.alloc(&d, (size_t)std::max<int64_t>(count, 1));
    if (e == cudaSuccess) e = cudaMemcpyAsync(d, src, sizeof(T) * count, cudaMemcpyHostToDevice, stream);
    *dst = d;
    return e;
  };
  CUDA_TRY(up(&sp->row_ptr, cfg->row_ptr, s + 1));
  CUDA_TRY(up(&sp->row_cum, cfg->row_cum, s));
  CUDA_TRY(up(&sp->row_scale, cfg->row_scale, s));
  if (cols) {
    CUDA_TRY(up(&sp->col_ptr, cfg->col_ptr, t + 1));
    CUDA_TRY(up(&sp->col_cum, cfg->col_cum, t));
    if (cfg->col_scale) CUDA_TRY(up(&sp->col_scale, cfg->col_scale, t));
  }
  if (dsbgs) {
    const int64_t total = cfg->dsbgs_off[t];
    CUDA_TRY(up(&sp->d_off, cfg->dsbgs_off, t + 1));
    CUDA_TRY(up(&sp->d_cum, cfg->dsbgs_cum, total));
    CUDA_TRY(up(&sp->d_total, cfg->dsbgs_total, t));
    CUDA_TRY(up(&sp->d_alive, cfg->dsbgs_alive, total));
    CUDA_TRY(up(&sp->d_scale, cfg->dsbgs_scale, s * t));
  }
  if (cfg->picks && cfg->max_iters > 0) CUDA_TRY(up(&sp->picks, cfg->picks, 2 * cfg->max_iters));
  return REBK_OK;
}

// DSBGS tables: offsets monotone from 0, alive indices in range, every
// scale finite and positive where the conditional can pick it
int check_dsbgs(const rebk_cfg* cfg) {
  const int64_t s = cfg->n_row_blocks, t = cfg->n_col_blocks;
  if (!cfg->dsbgs_off || !cfg->dsbgs_cum || !cfg->dsbgs_total || !cfg->dsbgs_alive || !cfg->dsbgs_scale)
    return fail(REBK_EINVAL, "dsbgs needs its joint-sampler tables (rebk_cfg.dsbgs_*)");
  if (cfg->dsbgs_off[0] != 0) return fail(REBK_EINVAL, "dsbgs_off[0] must be 0");
  for (int64_t j = 0; j < t; ++j) {
    if (cfg->dsbgs_off[j + 1] <= cfg->dsbgs_off[j])
      return fail(REBK_EINVAL, "column block %lld has no nonzero submatrix", (long long)j);
    for (int64_t e = cfg->dsbgs_off[j]; e < cfg->dsbgs_off[j + 1]; ++e) {
      const int32_t i = cfg->dsbgs_alive[e];
      if (i < 0 || i >= s) return fail(REBK_EINVAL, "dsbgs_alive entry out of range");
      if (!(cfg->dsbgs_scale[i * t + j] > 0.0)) return fail(REBK_EINVAL, "dsbgs scale must be positive");
    }
  }
  return REBK_OK;
}

int run_csr_impl(rebk_ctx* ctx, const rebk_cfg* cfg, const double* b_dev, const double* xs_dev, double* x_dev,
                 double* z_dev, cudaStream_t stream, rebk_trace* trace) {
  const bool extended = cfg->algorithm == REBK_ALGO_REBK || cfg->algorithm == REBK_ALGO_REK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  // u and r staged in shared memory when the largest blocks fit (REBK_CSR_STAGE=0: gathers from L2)
  const bool dsbgs_alg = cfg->algorithm == REBK_ALGO_DSBGS;
  int su_cap = extended ? ((max_block(cfg->n_col_blocks, cfg->col_ptr) + 1) & ~1) : 0;
  int sr_cap = (max_block(cfg->n_row_blocks, cfg->row_ptr) + 1) & ~1;
  if (env_int("REBK_CSR_STAGE", 1) == 0) su_cap = sr_cap = 0;
  if ((size_t)su_cap * 8 > kCsrStageBytesMax / 2) su_cap = 0;
  if ((size_t)(su_cap + sr_cap) * 8 > kCsrStageBytesMax) sr_cap = 0;
  (void)dsbgs_alg;
  int occ = 0;
  CUDA_TRY(csr_kernel_occupancy((size_t)(su_cap + sr_cap) * 8, &occ));
  int G = cfg->grid_ctas > 0 ? cfg->grid_ctas : grid_override();
  if (G <= 0) G = (int)std::min<int64_t>(std::max<int64_t>(1, (ctx->nnz + 8191) / 8192), (int64_t)ctx->sm_count);
  G = std::max(1, std::min(G, occ * ctx->sm_count));
  CsrSegPlan* sp = nullptr;
  int rc = build_seg_plan(ctx, cfg, extended, G, &sp);
  if (rc) return rc;

  DevArena arena;
  arena.stream = stream;
  const bool dsbgs = cfg->algorithm == REBK_ALGO_DSBGS;
  const int64_t s = cfg->n_row_blocks, t = (extended || dsbgs) ? cfg->n_col_blocks : 0;
  SampleParams smp{};
  rc = upload_sampler(arena, cfg, extended, extended || dsbgs, stream, &smp);
  if (rc) return rc;
  const int nJ_max = t > 0 ? max_block(t, cfg->col_ptr) : 1;
  const int nI_max = max_block(s, cfg->row_ptr);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(cfg->max_iters, (int64_t)1 << 20));
  Plan* d_plan;
  double *d_u, *d_r, *d_errpart, *d_res = nullptr, *d_errs = nullptr;
  Control* d_ctl;
  CUDA_TRY(arena.alloc(&d_plan, chunk));
  CUDA_TRY(arena.alloc(&d_u, std::max(nJ_max, 1)));
  CUDA_TRY(arena.alloc(&d_r, std::max(nI_max, 1)));
  CUDA_TRY(arena.alloc(&d_errpart, G));
  if (cfg->stop_mode == REBK_STOP_RESIDUAL_PROXY) CUDA_TRY(arena.alloc(&d_res, ctx->m));
  const int64_t errs_cap = (cfg->record_errors && trace && trace->errors) ? trace->errors_cap : 0;
  if (errs_cap > 0) CUDA_TRY(arena.alloc(&d_errs, errs_cap));
  CUDA_TRY(arena.alloc(&d_ctl, 1));
  CUDA_TRY(cudaMemsetAsync(d_ctl, 0, sizeof(Control), stream));
  long long* d_prof = nullptr;
  if (env_int("REBK_PROF", 0) == 1) {
    CUDA_TRY(arena.alloc(&d_prof, (size_t)G * 16));
    CUDA_TRY(cudaMemsetAsync(d_prof, 0, (size_t)G * 16 * 8, stream));
  }

  CsrParams p{};
  p.m = (int32_t)ctx->m;
  p.n = (int32_t)ctx->n;
  p.csr_ptr = ctx->csr_ptr;
  p.csr_col = ctx->csr_col;
  p.csr_val = ctx->csr_val;
  p.csc_ptr = ctx->csc_ptr;
  p.csc_row = ctx->csc_row;
  p.csc_val = ctx->csc_val;
  p.cseg_off = sp->cseg_off;
  p.cseg_row = sp->cseg_row;
  p.cseg_ptr = sp->cseg_ptr;
  p.cval = sp->cval;
  p.ccol = sp->ccol;
  p.cseg_cta = sp->cseg_cta;
  p.rseg_off = sp->rseg_off;
  p.rseg_col = sp->rseg_col;
  p.rseg_ptr = sp->rseg_ptr;
  p.rval = sp->rval;
  p.rrow = sp->rrow;
  p.rseg_cta = sp->rseg_cta;
  p.b = b_dev;
  p.xs = xs_dev;
  p.x = x_dev;
  p.z = z_dev;
  p.u = d_u;
  p.r = d_r;
  p.errpart = d_errpart;
  p.res = d_res;
  p.errs = d_errs;
  p.errs_cap = errs_cap;
  p.plan = d_plan;
  p.ctl = d_ctl;
  p.extended = extended;
  p.stop_mode = cfg->stop_mode;
  p.tol = cfg->tol;
  p.stride = cfg->check_stride;
  p.max_iters = cfg->max_iters;
  p.res_scale = cfg->residual_scale > 0.0 ? cfg->residual_scale : 1.0;
  p.record = errs_cap > 0;
  p.nonfinite_stop = cfg->nonfinite_stop;
  p.dsbgs = dsbgs;
  p.l2_prefetch = env_int("REBK_CSR_PF", 1);
  p.specialize = env_int("REBK_CSR_SPEC", 1);
  p.su_cap = su_cap;
  p.sr_cap = sr_cap;
  p.prof = d_prof;

  cudaEvent_t ev0, ev1;
  CUDA_TRY(cudaEventCreate(&ev0));
  CUDA_TRY(cudaEventCreate(&ev1));
  cudaError_t err = cudaEventRecord(ev0, stream);
  int64_t k = 1;
  do {
    const int64_t count = std::min(chunk, cfg->max_iters - k + 1);
    if (err == cudaSuccess) err = launch_sample_plan(smp, k, count, d_plan, nullptr, stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(&d_ctl->bar, 0, sizeof(unsigned long long), stream);
    p.k_begin = k;
    p.k_end = k + count - 1;
    if (err == cudaSuccess) err = launch_csr(p, G, stream);
    k += std::max<int64_t>(count, 1);
    if (err == cudaSuccess && k <= cfg->max_iters) {
      int32_t done = 0;
      err = cudaMemcpyAsync(&done, &d_ctl->done, sizeof done, cudaMemcpyDeviceToHost, stream);
      if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
      if (done) break;
    }
  } while (err == cudaSuccess && k <= cfg->max_iters);
  if (err == cudaSuccess) err = cudaEventRecord(ev1, stream);
  Control ctl{};
  if (err == cudaSuccess) err = cudaMemcpyAsync(&ctl, d_ctl, sizeof ctl, cudaMemcpyDeviceToHost, stream);
  if (err == cudaSuccess && errs_cap > 0)
    err = cudaMemcpyAsync(trace->errors, d_errs, errs_cap * sizeof(double), cudaMemcpyDeviceToHost, stream);
  if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
  float ms = 0.f;
  if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (err != cudaSuccess) return fail(REBK_ECUDA, "sparse REBK run failed: %s", cudaGetErrorString(err));
  if (d_prof) {
    std::vector<long long> h((size_t)G * 16);
    cudaMemcpy(h.data(), d_prof, h.size() * 8, cudaMemcpyDeviceToHost);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx->device);
    const double it = (double)std::max<int64_t>(1, ctl.iters);
    fprintf(stderr, "[rebk prof] path=csr G=%d iters=%lld loop=%.3f ms (%.3f us/iter); mark mean max\n", G,
            (long long)ctl.iters, ms, 1e3 * ms / it);
    print_prof(h, G, G, khz, it);
  }
  if (trace) {
    trace->iters = ctl.iters;
    trace->converged = ctl.converged;
    trace->has_error = ctl.has_error;
    trace->final_error = ctl.final_error;
    trace->loop_ms = ms;
    trace->n_checks = ctl.n_checks;
    trace->grid_ctas = G;
    trace->kernel_path = 3;
    trace->nonfinite_at = ctl.nonfinite_at - 1;
  }
  if (ctl.nonfinite_at && cfg->nonfinite_stop)
    return fail(REBK_ENONFINITE, "non-finite error at the check of iteration %lld", (long long)(ctl.nonfinite_at - 1));
  return REBK_OK;
}

// REBK_HOST_TIMING=1: host wall-clock marks of one dense run's phases (stderr)
struct HostMarks {
  bool on = false;
  std::chrono::steady_clock::time_point t0, last;
  HostMarks() {
    const char* e = getenv("REBK_HOST_TIMING");
    on = e && atoi(e) != 0;
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[rebk host] %-28s +%8.3f ms (total %8.3f ms)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(),
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

// internal: the clustered kernels could not run (cooperative cluster launch
// refused, or launched without their clusters); nothing was written yet
constexpr int kRetryGeneral = 100;

int run_device_impl_once(rebk_ctx* ctx, const rebk_cfg* cfg, const double* b_dev, const double* xs_dev,
                         double* x_dev, double* z_dev, cudaStream_t stream, rebk_trace* trace, bool force_general) {
  const bool extended = cfg->algorithm == REBK_ALGO_REBK || cfg->algorithm == REBK_ALGO_REK;
  const bool dsbgs = cfg->algorithm == REBK_ALGO_DSBGS;
  if (cfg->algorithm < 0 || cfg->algorithm > 4) return fail(REBK_EINVAL, "unknown algorithm %d", cfg->algorithm);
  if (cfg->stop_mode < 0 || cfg->stop_mode > 2) return fail(REBK_EINVAL, "unknown stopping mode %d", cfg->stop_mode);
  if (cfg->stop_mode != REBK_STOP_MAX_ITERS_ONLY && !(cfg->tol > 0.0)) return fail(REBK_EINVAL, "tol must be positive");
  if (cfg->check_stride < 1) return fail(REBK_EINVAL, "check_stride must be at least 1");
  if (cfg->max_iters < 0) return fail(REBK_EINVAL, "max_iters must be nonnegative");
  if (cfg->stop_mode == REBK_STOP_ORACLE_ERROR && !xs_dev)
    return fail(REBK_EINVAL, "oracle_error stopping needs a problem with x_star");
  if (!b_dev || !x_dev || (extended && !z_dev)) return fail(REBK_EINVAL, "missing b / x / z buffer");
  int rc = check_partition("row", cfg->n_row_blocks, cfg->row_ptr, cfg->row_cum, cfg->row_scale, ctx->m);
  if (rc) return rc;
  if (extended || dsbgs) {
    rc = check_partition("col", cfg->n_col_blocks, cfg->col_ptr, cfg->col_cum, dsbgs ? cfg->col_cum : cfg->col_scale,
                         ctx->n);
    if (rc) return rc;
  }
  if (dsbgs && (rc = check_dsbgs(cfg)) != 0) return rc;
  if (ctx->m > INT32_MAX || ctx->n > INT32_MAX) return fail(REBK_EINVAL, "matrix dimension exceeds 2^31");
  if (ctx->kind == 2) return fail(REBK_EINVAL, "fp32 contexts run through rebk_run_mrhs");
  if (ctx->kind == 1) return run_csr_impl(ctx, cfg, b_dev, xs_dev, x_dev, z_dev, stream, trace);

  CUDA_TRY(cudaSetDevice(ctx->device));
  HostMarks hm;

  // geometry: find the largest grid that is co-resident with our smem need
  int G0 = choose_grid(ctx, cfg, 1 << 20);
  Geometry geo = plan_geometry(ctx, cfg, G0, extended);
  int occ = 0;
  CUDA_TRY(dense_kernel_occupancy(geo.smem_bytes, &occ));
  if (occ < 1) return fail(REBK_EINVAL, "problem too large for one CTA's shared memory (%zu bytes)", geo.smem_bytes);
  if (G0 > occ * ctx->sm_count) {
    geo = plan_geometry(ctx, cfg, occ * ctx->sm_count, extended);
  }
  hm.mark("geometry + occupancy");
  // fast path: clustered kernel (oracle_error / max_iters_only, TMA-able tiles,
  // at least one full cluster).  The choice depends only on the problem shape,
  // partitions and stopping mode, so repeated runs take the same path.
  // residual_proxy on the fast kernels: they iterate in chunks of
  // check_stride in max_iters_only mode, and stand-alone residual-check
  // kernels run between the chunks (launch_residual_check); worth it once a
  // check covers enough iterations (REBK_RES_MIN_STRIDE, default 8)
  const bool res_mode = cfg->stop_mode == REBK_STOP_RESIDUAL_PROXY;
  const bool res_chunks_ok = res_mode && cfg->check_stride >= env_int("REBK_RES_MIN_STRIDE", 8);
  FastGeometry fg;
  bool use_fast = false;
  CUtensorMap tm_ct, tm_rt;
  {
    const int CS = kClusterCS;  // the clustered kernels' compile-time cluster shape
    const bool aligned = (ctx->lda % 2 == 0) && ((uintptr_t)ctx->A % 16 == 0);
    // TMA boxes start on 16-byte aligned columns: the clustered kernels need
    // even column-block starts (the streaming kernel handles odd ones)
    const bool even_cols = !extended || blocks_even(cfg->n_col_blocks, cfg->col_ptr);
    if (!force_general && !dsbgs && env_int("REBK_NO_FAST", 0) == 0 && (!res_mode || res_chunks_ok) && aligned && even_cols && CS >= 1 &&
        G0 >= CS && encode_fn() != nullptr) {
      // (a finer grid for small problems was measured and not adopted: C1 on
      // 40-88 CTAs instead of 16 runs 6.7 instead of 7.9 us per iteration, but
      // its end-to-end rate was more variable and on average lower (56-67k
      // against a steady 65-68k iters/s); profiles/r02_c1_grid_sweep.txt.
      // REBK_GRID selects it.)
      const int Gf = G0;
      int NC = std::max(1, Gf / CS);
      for (int attempt = 0; attempt < 3 && NC >= 1; ++attempt) {
        fg = fast_geometry(ctx, cfg, extended, NC, CS);
        if (!fg.ok) break;
        int maxc = 0;
        if (fast_max_clusters(CS, fg.smem_bytes, &maxc) != cudaSuccess || maxc < 1) {
          fg.ok = false;
          cudaGetLastError();
          break;
        }
        if (NC <= maxc) break;
        NC = maxc;
      }
      if (fg.ok && fg.NC == NC) {
        use_fast = encode_box(&tm_ct, ctx, fg.ct_box_w, fg.ct_box_h) &&
                   encode_box(&tm_rt, ctx, fg.rt_box_w, fg.rt_box_h);
      }
    }
  }
  hm.mark("fast-path probe");
  // split path: column and row sweeps on two concurrent CTA groups
  // (rebk_dense_split.cu); needs a column sweep and oracle/no stopping
  bool use_split = false;
  int split_ncc = 0;
  const int split_xmode = env_int("REBK_SPLIT_XMODE", 0);  // bit 0/1: column/row group exchanges gather all
  const int split_pieces = std::max(1, std::min(2, env_int("REBK_SPLIT_PIECES", 2)));
  if (use_fast && extended && env_int("REBK_SPLIT", 1) != 0 && fg.NC >= 2) {
    const int NC = fg.NC, CS = fg.CS;
    const double colb = (double)ctx->m * max_block(cfg->n_col_blocks, cfg->col_ptr);
    const double rowb = (double)ctx->n * max_block(cfg->n_row_blocks, cfg->row_ptr);
    int ncc = (int)(NC * colb / (colb + rowb) + 0.5);
    ncc = env_int("REBK_SPLIT_NCC", ncc);
    ncc = std::max(1, std::min(NC - 1, ncc));
    FastGeometry sg = split_geometry(ctx, cfg, NC, CS, ncc, split_xmode, split_pieces);
    int maxc = 0;
    if (sg.ok && split_max_clusters(CS, sg.smem_bytes, &maxc) == cudaSuccess && maxc >= NC &&
        encode_box(&tm_ct, ctx, sg.ct_box_w, sg.ct_box_h) && encode_box(&tm_rt, ctx, sg.rt_box_w, sg.rt_box_h)) {
      fg = sg;
      use_split = true;
      split_ncc = ncc;
    } else {
      cudaGetLastError();
      // restore the fused path's tensor maps
      use_fast = encode_box(&tm_ct, ctx, fg.ct_box_w, fg.ct_box_h) && encode_box(&tm_rt, ctx, fg.rt_box_w, fg.rt_box_h);
    }
  }
  hm.mark("split-path probe");
  // streaming path: blocks whose per-CTA slices the general kernel cannot
  // stage in shared memory (C3) stream through a TMA ring instead
  bool use_stream = false;
  StreamGeometry stg;
  CUtensorMap tm_sc, tm_sr;
  const int stream_env = env_int("REBK_STREAM", 1);  // 0 off, 1 when the general kernel cannot stage, 2 always
  if (!use_fast && !dsbgs && stream_env != 0 && (!res_mode || res_chunks_ok) &&
      (ctx->lda % 2 == 0) && ((uintptr_t)ctx->A % 16 == 0) && encode_fn() != nullptr &&
      (stream_env == 2 || tiles_exceed_smem(geo, extended))) {
    stg = stream_geometry(ctx, cfg, std::min(G0, ctx->sm_count), extended);
    int occs = 0;
    if (stg.ok && stream_kernel_occupancy(stg.smem_bytes, &occs) == cudaSuccess && occs >= 1 &&
        (!extended || encode_box(&tm_sc, ctx, stg.cw, stg.ch)) && encode_box(&tm_sr, ctx, stg.rw, stg.rh)) {
      use_stream = true;
      if (!extended) tm_sc = tm_sr;
    }
    cudaGetLastError();
  }
  const int G = use_fast ? fg.G : (use_stream ? stg.G : geo.G);

  DevArena arena;
  arena.stream = stream;
  hm.mark("path selection");
  SampleParams sp{};
  rc = upload_sampler(arena, cfg, extended, extended || dsbgs, stream, &sp);
  if (rc) return rc;
  const bool res_fast = res_mode && (use_fast || use_split || use_stream);
  const int64_t chunk = res_fast ? cfg->check_stride
                                 : std::max<int64_t>(1, std::min<int64_t>(cfg->max_iters, (int64_t)1 << 20));
  Plan* d_plan;
  double *d_upart, *d_rpart, *d_u, *d_r, *d_errpart, *d_res = nullptr, *d_errs = nullptr;
  Control* d_ctl;
  CUDA_TRY(arena.alloc(&d_plan, chunk));
  CUDA_TRY(arena.alloc(&d_upart, (size_t)std::max(geo.nJ_max, 1) * G));
  CUDA_TRY(arena.alloc(&d_rpart, (size_t)std::max(geo.nI_max, 1) * G));
  CUDA_TRY(arena.alloc(&d_u, std::max(geo.nJ_max, 1)));
  CUDA_TRY(arena.alloc(&d_r, std::max(geo.nI_max, 1)));
  CUDA_TRY(arena.alloc(&d_errpart, G));
  LLWord* d_zring = nullptr;
  double* d_zhist = nullptr;
  SplitShared* d_sh = nullptr;
  const int split_D = std::max(2, env_int("REBK_SPLIT_RING", 16)), split_H = split_D + 4;
  if (use_split) {
    CUDA_TRY(arena.alloc(&d_zring, (size_t)split_D * fg.nI_max));
    CUDA_TRY(cudaMemsetAsync(d_zring, 0, (size_t)split_D * fg.nI_max * sizeof(LLWord), stream));
    CUDA_TRY(arena.alloc(&d_zhist, (size_t)split_H * ctx->m));
    CUDA_TRY(arena.alloc(&d_sh, 1));
    CUDA_TRY(cudaMemsetAsync(d_sh, 0, sizeof(SplitShared), stream));
  }
  LLWord *d_cpu = nullptr, *d_cpr = nullptr;
  if (use_fast) {
    // two slots each (exchange sequence parity)
    CUDA_TRY(arena.alloc(&d_cpu, 2 * (size_t)fg.NC * (fg.nJ_max + 1)));
    CUDA_TRY(arena.alloc(&d_cpr, 2 * (size_t)fg.NC * (2 * fg.nI_max + 1)));
    CUDA_TRY(cudaMemsetAsync(d_cpu, 0, 2 * (size_t)fg.NC * (fg.nJ_max + 1) * sizeof(LLWord), stream));
    CUDA_TRY(cudaMemsetAsync(d_cpr, 0, 2 * (size_t)fg.NC * (2 * fg.nI_max + 1) * sizeof(LLWord), stream));
  }
  if (cfg->stop_mode == REBK_STOP_RESIDUAL_PROXY) CUDA_TRY(arena.alloc(&d_res, ctx->m));
  // streaming kernel: z before the latest column sweep (its column sweep runs one step ahead of the row sweep)
  double* d_zprev = nullptr;
  if (use_stream && extended) CUDA_TRY(arena.alloc(&d_zprev, ctx->m));
  double *d_rpart_chk = nullptr, *d_colsq = nullptr;
  if (res_fast) {
    CUDA_TRY(arena.alloc(&d_rpart_chk, residual_check_part_len((int)ctx->m, (int)ctx->n)));
    CUDA_TRY(arena.alloc(&d_colsq, ctx->n));
  }
  const int64_t errs_cap = (cfg->record_errors && trace && trace->errors) ? trace->errors_cap : 0;
  if (errs_cap > 0) CUDA_TRY(arena.alloc(&d_errs, errs_cap));
  CUDA_TRY(arena.alloc(&d_ctl, 1));
  // REBK_TRACE=n: globaltimer stamps of the split exchanges for iterations
  // [REBK_TRACE_K0, +n), written raw to REBK_TRACE_FILE (tools/trace_split.py)
  const int trace_n = env_int("REBK_TRACE", 0);
  const int64_t trace_k0 = env_int("REBK_TRACE_K0", 2000);
  unsigned long long* d_trace = nullptr;
  if (trace_n > 0 && use_split) {
    CUDA_TRY(arena.alloc(&d_trace, (size_t)trace_n * G * 8));
    CUDA_TRY(cudaMemsetAsync(d_trace, 0, (size_t)trace_n * G * 8 * 8, stream));
  }
  const char* prof_env = getenv("REBK_PROF");
  long long* d_prof = nullptr;
  if (prof_env && prof_env[0] == '1') {
    CUDA_TRY(arena.alloc(&d_prof, (size_t)G * 16));
    CUDA_TRY(cudaMemsetAsync(d_prof, 0, (size_t)G * 16 * 8, stream));
  }
  CUDA_TRY(cudaMemsetAsync(d_ctl, 0, sizeof(Control), stream));

  DenseParams p{};
  p.A = ctx->A;
  p.lda = ctx->lda;
  p.m = (int32_t)ctx->m;
  p.n = (int32_t)ctx->n;
  p.b = b_dev;
  p.xs = xs_dev;
  p.x = x_dev;
  p.z = z_dev;
  p.upart = d_upart;
  p.rpart = d_rpart;
  p.u = d_u;
  p.r = d_r;
  p.errpart = d_errpart;
  p.res = d_res;
  p.errs = d_errs;
  p.errs_cap = errs_cap;
  p.plan = d_plan;
  p.ctl = d_ctl;
  p.prof = d_prof;
  p.extended = extended;
  p.stop_mode = cfg->stop_mode;
  p.tol = cfg->tol;
  p.stride = cfg->check_stride;
  p.max_iters = cfg->max_iters;
  p.res_scale = cfg->residual_scale > 0.0 ? cfg->residual_scale : 1.0;
  p.record = errs_cap > 0;
  p.nonfinite_stop = cfg->nonfinite_stop;
  p.dsbgs = dsbgs;
  if (res_fast) {  // the kernels iterate; the checks are separate launches
    p.stop_mode = REBK_STOP_MAX_ITERS_ONLY;
    p.max_iters = INT64_MAX;
  }
  p.nJ_max = geo.nJ_max;
  p.nI_max = geo.nI_max;
  p.nR_max = geo.nR_max;
  p.nC_max = geo.nC_max;
  p.ct_ld = geo.ct_ld;
  p.rt_ld = geo.rt_ld;
  p.stage_ct = geo.stage_ct;
  p.stage_rt = geo.stage_rt;
  p.ct_off = geo.ct_off;
  p.rt_off = geo.rt_off;
  p.vec_off = geo.vec_off;

  FastParams fpar{};
  if (use_fast) {
    p.nJ_max = fg.nJ_max;
    p.nI_max = fg.nI_max;
    p.nR_max = fg.nR_max;
    p.nC_max = fg.nC_max;
    p.ct_off = fg.ct_off;
    p.rt_off = fg.rt_off;
    p.vec_off = fg.vec_off;
    p.stage_ct = p.stage_rt = 1;
    fpar.cpart_u = d_cpu;
    fpar.cpart_r = d_cpr;
    fpar.stride_u = fg.nJ_max + 1;
    fpar.stride_r = 2 * fg.nI_max + 1;
    fpar.ct_box_w = fg.ct_box_w;
    fpar.ct_box_h = fg.ct_box_h;
    fpar.rt_box_w = fg.rt_box_w;
    fpar.rt_box_h = fg.rt_box_h;
    fpar.pad_nC = fg.pad_nC;
    fpar.pad_nR = fg.pad_nR;
    fpar.pad_ne = fg.pad_ne;
    fpar.pad_in = fg.pad_in;
    fpar.pad_cin = fg.pad_cin;
    fpar.cluster_size = fg.CS;
  }
  cudaEvent_t ev0, ev1;
  CUDA_TRY(cudaEventCreate(&ev0));
  CUDA_TRY(cudaEventCreate(&ev1));
  cudaError_t err = cudaEventRecord(ev0, stream);
  hm.mark("workspace + uploads");
  auto res_check = [&](int64_t kc) -> cudaError_t {
    return launch_residual_check(ctx->A, ctx->lda, (int)ctx->m, (int)ctx->n, x_dev, b_dev, extended ? z_dev : nullptr,
                                 d_res, d_rpart_chk, d_colsq, cfg->residual_scale > 0.0 ? cfg->residual_scale : 1.0,
                                 cfg->tol, cfg->nonfinite_stop, errs_cap > 0, d_errs, errs_cap, kc, d_ctl, stream);
  };
  if (res_fast && err == cudaSuccess) err = res_check(0);  // check(0), solvers.py:444
  int64_t k = 1;
  int chunks_since_sync = 0;
  do {
    const int64_t count = std::min(chunk, cfg->max_iters - k + 1);
    if (err == cudaSuccess) err = launch_sample_plan(sp, k, count, d_plan, nullptr, stream);
    if (err == cudaSuccess) err = cudaMemsetAsync(&d_ctl->bar, 0, sizeof(unsigned long long), stream);
    p.k_begin = k;
    p.k_end = k + count - 1;
    if (err == cudaSuccess) {
      if (use_split) {
        fpar.d = p;
        SplitParams spar{};
        spar.f = fpar;
        spar.ncc = split_ncc;
        spar.ring = split_D;
        spar.hist = split_H;
        spar.zr_stride = fg.nI_max;
        spar.zring = d_zring;
        spar.zhist = d_zhist;
        spar.sh = d_sh;
        spar.vec_off_c = fg.vec_off_c;
        spar.vec_off_r = fg.vec_off_r;
        spar.xmode = split_xmode;
        spar.pieces = fg.pieces;
        spar.trace = d_trace;
        spar.trace_k0 = trace_k0;
        spar.trace_n = trace_n;
        err = launch_dense_split(spar, tm_ct, tm_rt, G, fg.CS, fg.smem_bytes, stream);
      } else if (use_fast) {
        fpar.d = p;
        err = launch_dense_fast(fpar, tm_ct, tm_rt, G, fg.CS, fg.smem_bytes, stream);
      } else if (use_stream) {
        StreamParams spar{};
        spar.d = p;
        spar.stages = stg.NS;
        spar.stage_doubles = stg.SD;
        spar.cw = stg.cw;
        spar.ch = stg.ch;
        spar.rw = stg.rw;
        spar.rh = stg.rh;
        spar.lc = stg.lc;
        spar.lr = stg.lr;
        spar.pad_nC = stg.pad_nC;
        spar.pad_nR = stg.pad_nR;
        spar.pad_nJ = stg.pad_nJ;
        spar.pad_nI = stg.pad_nI;
        spar.l2hint = env_int("REBK_STREAM_L2HINT", 1);
        spar.reverse = env_int("REBK_STREAM_REV", 1);
        spar.prefetch = env_int("REBK_STREAM_PF", 0);
        spar.pfence = env_int("REBK_STREAM_PFENCE", 0);
        spar.dbg = env_int("REBK_STREAM_DBG", 0);
        spar.order = env_int("REBK_STREAM_ORDER", 0);
  spar.tail = stream_tail(ctx, ctx->m, stg.nJ_max, stg.nI_max, extended);
        spar.zprev = d_zprev;
        err = launch_dense_stream(spar, tm_sc, tm_sr, G, stg.smem_bytes, stream);
      } else {
        err = launch_dense(p, G, geo.smem_bytes, stream);
      }
      // the spin-barrier kernels only ever run as cooperative launches (all
      // CTAs co-resident); if the cooperative cluster launch is refused, the
      // run goes to the general kernel instead of a grid that could hang
      if (err != cudaSuccess && (use_fast || use_split) && k == 1) {
        cudaGetLastError();
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        return kRetryGeneral;
      }
    }
    k += std::max<int64_t>(count, 1);
    if (res_fast && err == cudaSuccess) {
      const int64_t ke = k - 1;  // state of iteration ke: a check on stride, and the for-else final check
      if (ke % cfg->check_stride == 0 || ke == cfg->max_iters) err = res_check(ke);
    }
    // converged runs stop early: the host looks at the device flag after every
    // chunk (every 32 chunks in residual-check mode, whose launches are short
    // and return at once once the flag is set)
    if (err == cudaSuccess && k <= cfg->max_iters && (!res_fast || ++chunks_since_sync >= 32)) {
      chunks_since_sync = 0;
      int32_t done = 0;
      err = cudaMemcpyAsync(&done, &d_ctl->done, sizeof done, cudaMemcpyDeviceToHost, stream);
      if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
      if (done) break;
    }
  } while (err == cudaSuccess && k <= cfg->max_iters);
  if (err == cudaSuccess) err = cudaEventRecord(ev1, stream);
  hm.mark("launch loop (async)");
  Control ctl{};
  if (err == cudaSuccess) err = cudaMemcpyAsync(&ctl, d_ctl, sizeof ctl, cudaMemcpyDeviceToHost, stream);
  if (err == cudaSuccess && errs_cap > 0) {
    const int64_t nrec = errs_cap;
    err = cudaMemcpyAsync(trace->errors, d_errs, nrec * sizeof(double), cudaMemcpyDeviceToHost, stream);
  }
  if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
  float ms = 0.f;
  if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (err != cudaSuccess) return fail(REBK_ECUDA, "REBK run failed: %s", cudaGetErrorString(err));
  hm.mark("sync + control readback");
  // launched without its clusters (e.g. replayed by a profiler that drops
  // the cluster shape): every CTA refused before touching x / z, so the run
  // is repeated on the general kernel
  if (ctl.fault) return kRetryGeneral;
  if (d_trace) {
    std::vector<unsigned long long> h((size_t)trace_n * G * 8);
    cudaMemcpy(h.data(), d_trace, h.size() * 8, cudaMemcpyDeviceToHost);
    const char* fn = getenv("REBK_TRACE_FILE");
    FILE* f = fopen(fn ? fn : "rebk_trace.bin", "wb");
    if (f) {
      const int32_t hdr[4] = {trace_n, G, split_ncc * fg.CS, fg.CS};
      fwrite(hdr, sizeof hdr, 1, f);
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  if (d_prof) {
    std::vector<long long> h((size_t)G * 16);
    cudaMemcpy(h.data(), d_prof, h.size() * 8, cudaMemcpyDeviceToHost);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx->device);
    const double it = (double)std::max<int64_t>(1, ctl.iters);
    fprintf(stderr, "[rebk prof] path=%s ncc=%d ",
            use_split ? "split" : (use_fast ? "fast(coop)" : (use_stream ? "stream" : "v1")),
            split_ncc);
    fprintf(stderr, "[rebk prof] G=%d iters=%lld loop=%.3f ms (%.3f us/iter); per-iteration us: mark mean max\n", G,
            (long long)ctl.iters, ms, 1e3 * ms / it);
    print_prof(h, G, use_split ? split_ncc * fg.CS : G, khz, it);
  }
  // residual checks between chunks: a run that never stopped ends at max_iters
  // (the for-else of run(), solvers.py:459-464)
  if (res_fast && !ctl.converged && !(ctl.nonfinite_at && cfg->nonfinite_stop)) ctl.iters = cfg->max_iters;
  if (trace) {
    trace->iters = ctl.iters;
    trace->converged = ctl.converged;
    trace->has_error = ctl.has_error;
    trace->final_error = ctl.final_error;
    trace->loop_ms = ms;
    trace->n_checks = ctl.n_checks;
    trace->grid_ctas = G;
    trace->kernel_path = use_split ? 6 : (use_fast ? 2 : (use_stream ? 7 : 0));
    trace->nonfinite_at = ctl.nonfinite_at - 1;
  }
  if (ctl.nonfinite_at && cfg->nonfinite_stop)
    return fail(REBK_ENONFINITE, "non-finite error at the check of iteration %lld", (long long)(ctl.nonfinite_at - 1));
  return REBK_OK;
}

int run_device_impl(rebk_ctx* ctx, const rebk_cfg* cfg, const double* b_dev, const double* xs_dev,
                    double* x_dev, double* z_dev, cudaStream_t stream, rebk_trace* trace) {
  int rc = run_device_impl_once(ctx, cfg, b_dev, xs_dev, x_dev, z_dev, stream, trace, false);
  if (rc == kRetryGeneral) rc = run_device_impl_once(ctx, cfg, b_dev, xs_dev, x_dev, z_dev, stream, trace, true);
  if (rc == kRetryGeneral) rc = fail(REBK_ECUDA, "the general kernel refused its launch");
  return rc;
}


// ---- row-sharded streaming path (rebk_shard_stream_kernel) -----
// Exchange buffer of one rank: inbox_u [2][P][nJ_cap], inbox_x [2][P][n_cap],
// flags [2][2][P][Gr] (layout documented at RankXchg).
size_t xchg_bytes(int P, int64_t nJ_cap, int64_t n_cap, int Gr) {
  return sizeof(double) * (size_t)(2 * P * nJ_cap + 2 * P * n_cap) + sizeof(unsigned long long) * (size_t)(4 * P * Gr);
}
void xchg_carve(char* base, int P, int64_t nJ_cap, int64_t n_cap, double** iu, double** ix, unsigned long long** fl) {
  *iu = (double*)base;
  *ix = *iu + 2 * P * nJ_cap;
  *fl = (unsigned long long*)(*ix + 2 * P * n_cap);
}

struct ShardLaunch {
  int vranks = 1, P = 1, rank = 0, Gr = 0;
  const int64_t* rows = nullptr;    // [vranks] local rows of each (virtual) rank
  const int64_t* ranges = nullptr;  // host [vranks][s][2]
  char* xbuf[kMaxRanks] = {};       // exchange buffer of every rank, as seen from this GPU
  int64_t nJ_cap = 0, n_cap = 0;
  unsigned long long seq_base = 0;
};

int shard_stream_impl(rebk_ctx* ctx, const rebk_cfg* cfg, ShardLaunch& L, const double* b_dev, const double* xs_dev,
                      double* x_dev, double* z_dev, cudaStream_t stream, rebk_trace* trace) {
  const bool extended = cfg->algorithm == REBK_ALGO_REBK || cfg->algorithm == REBK_ALGO_REK;
  if (cfg->algorithm < 0 || cfg->algorithm > 3) return fail(REBK_EINVAL, "unknown algorithm %d", cfg->algorithm);
  if (cfg->stop_mode != REBK_STOP_ORACLE_ERROR && cfg->stop_mode != REBK_STOP_MAX_ITERS_ONLY)
    return fail(REBK_EINVAL, "the row-sharded path supports oracle_error and max_iters_only stopping");
  if (cfg->stop_mode == REBK_STOP_ORACLE_ERROR && !(cfg->tol > 0.0)) return fail(REBK_EINVAL, "tol must be positive");
  if (cfg->stop_mode == REBK_STOP_ORACLE_ERROR && !xs_dev)
    return fail(REBK_EINVAL, "oracle_error stopping needs a problem with x_star");
  if (cfg->check_stride < 1 || cfg->max_iters < 0) return fail(REBK_EINVAL, "bad check_stride / max_iters");
  if (!b_dev || !x_dev || (extended && !z_dev)) return fail(REBK_EINVAL, "missing b / x / z buffer");
  if (ctx->kind != 0) return fail(REBK_EINVAL, "the row-sharded path needs a dense fp64 context");
  if (L.vranks < 1 || L.vranks > kMaxRanks || L.P < 1 || L.P > kMaxRanks || L.rank < 0 || L.rank >= L.P ||
      (L.vranks > 1 && L.vranks != L.P))
    return fail(REBK_EINVAL, "bad rank layout (P = %d, rank = %d, vranks = %d; at most %d ranks)", L.P, L.rank,
                L.vranks, kMaxRanks);
  const int64_t s = cfg->n_row_blocks;
  if (s < 1 || !cfg->row_ptr) return fail(REBK_EINVAL, "row partition missing");
  int rc = check_partition("row", s, cfg->row_ptr, cfg->row_cum, cfg->row_scale, cfg->row_ptr[s]);
  if (rc) return rc;
  if (extended) {
    rc = check_partition("col", cfg->n_col_blocks, cfg->col_ptr, cfg->col_cum, cfg->col_scale, ctx->n);
    if (rc) return rc;
  }
  // every rank's local ranges: block b's rows are [lo, hi), consecutive, and
  // together they are the rank's rows; ranks stacked in the ctx for vranks > 1
  int64_t stacked = 0, m_max = 0, nI_loc = 1;
  for (int v = 0; v < L.vranks; ++v) {
    const int64_t* rg = L.ranges + (int64_t)v * 2 * s;
    int64_t pos = 0;
    for (int64_t b = 0; b < s; ++b) {
      if (rg[2 * b] != pos || rg[2 * b + 1] < pos || rg[2 * b + 1] - rg[2 * b] > cfg->row_ptr[b + 1] - cfg->row_ptr[b])
        return fail(REBK_EINVAL, "rank %d: local row ranges must be consecutive shares of the row blocks", v);
      pos = rg[2 * b + 1];
      nI_loc = std::max(nI_loc, rg[2 * b + 1] - rg[2 * b]);
    }
    if (pos != L.rows[v]) return fail(REBK_EINVAL, "rank %d: ranges cover %lld rows, the rank holds %lld", v,
                                      (long long)pos, (long long)L.rows[v]);
    stacked += L.rows[v];
    m_max = std::max(m_max, L.rows[v]);
  }
  if (stacked != ctx->m) return fail(REBK_EINVAL, "the ctx holds %lld rows, the ranks %lld", (long long)ctx->m,
                                     (long long)stacked);
  if (ctx->n > INT32_MAX || ctx->m > INT32_MAX) return fail(REBK_EINVAL, "matrix dimension exceeds 2^31");
  if ((ctx->lda % 2) != 0 || ((uintptr_t)ctx->A % 16) != 0 || encode_fn() == nullptr)
    return fail(REBK_EINVAL, "the row-sharded path needs a 16-byte aligned A with an even leading dimension");
  const int nJ_max = extended ? max_block(cfg->n_col_blocks, cfg->col_ptr) : 0;
  if (nJ_max > L.nJ_cap || ctx->n > L.n_cap) return fail(REBK_EINVAL, "exchange buffers too small for this problem");
  CUDA_TRY(cudaSetDevice(ctx->device));
  StreamGeometry stg = stream_geometry_dims(std::max<int64_t>(m_max, 1), ctx->n, (int)nI_loc, nJ_max,
                                            !extended || blocks_even(cfg->n_col_blocks, cfg->col_ptr), L.Gr, extended);
  int occ = 0;
  if (!stg.ok || stream_kernel_occupancy(stg.smem_bytes, &occ) != cudaSuccess || occ < 1)
    return fail(REBK_EINVAL, "row-sharded geometry does not fit shared memory");
  if (L.vranks * L.Gr > occ * ctx->sm_count)
    return fail(REBK_EINVAL, "%d ranks x %d CTAs are not co-resident on this GPU", L.vranks, L.Gr);
  CUtensorMap tm_c, tm_r;
  if (!(extended ? encode_box(&tm_c, ctx, stg.cw, stg.ch) : true) || !encode_box(&tm_r, ctx, stg.rw, stg.rh))
    return fail(REBK_ECUDA, "tensor map encoding failed");
  if (!extended) tm_c = tm_r;

  DevArena arena;
  arena.stream = stream;
  const int64_t t = extended ? cfg->n_col_blocks : 0;
  const int G = L.Gr;
  int64_t *d_row_ptr, *d_col_ptr = nullptr, *d_ranges;
  double *d_row_cum, *d_row_scale, *d_col_cum = nullptr, *d_col_scale = nullptr;
  CUDA_TRY(arena.alloc(&d_row_ptr, s + 1));
  CUDA_TRY(arena.alloc(&d_row_cum, s));
  CUDA_TRY(arena.alloc(&d_row_scale, s));
  CUDA_TRY(arena.alloc(&d_ranges, (size_t)L.vranks * 2 * s));
  CUDA_TRY(cudaMemcpyAsync(d_row_ptr, cfg->row_ptr, (s + 1) * 8, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(d_row_cum, cfg->row_cum, s * 8, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(d_row_scale, cfg->row_scale, s * 8, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(d_ranges, L.ranges, (size_t)L.vranks * 2 * s * 8, cudaMemcpyHostToDevice, stream));
  if (extended) {
    CUDA_TRY(arena.alloc(&d_col_ptr, t + 1));
    CUDA_TRY(arena.alloc(&d_col_cum, t));
    CUDA_TRY(arena.alloc(&d_col_scale, t));
    CUDA_TRY(cudaMemcpyAsync(d_col_ptr, cfg->col_ptr, (t + 1) * 8, cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(d_col_cum, cfg->col_cum, t * 8, cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(d_col_scale, cfg->col_scale, t * 8, cudaMemcpyHostToDevice, stream));
  }
  int32_t* d_picks = nullptr;
  if (cfg->picks && cfg->max_iters > 0) {
    CUDA_TRY(arena.alloc(&d_picks, 2 * cfg->max_iters));
    CUDA_TRY(cudaMemcpyAsync(d_picks, cfg->picks, 2 * cfg->max_iters * sizeof(int32_t), cudaMemcpyHostToDevice, stream));
  }
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(cfg->max_iters, (int64_t)1 << 20));
  Plan* d_plan;
  CUDA_TRY(arena.alloc(&d_plan, chunk));
  // per-rank workspace, identical layout at vr * ws_stride
  const int64_t nJw = std::max(nJ_max, 1), nIw = std::max<int64_t>(nI_loc, 1);
  const int64_t o_rpart = nJw * G, o_u = o_rpart + nIw * G, o_r = o_u + nJw, o_err = o_r + nIw;
  const int64_t ws_stride = (o_err + G + 1) & ~(int64_t)1;
  double* d_ws;
  CUDA_TRY(arena.alloc(&d_ws, (size_t)ws_stride * L.vranks));
  Control* d_ctl;
  CUDA_TRY(arena.alloc(&d_ctl, L.vranks));
  CUDA_TRY(cudaMemsetAsync(d_ctl, 0, sizeof(Control) * L.vranks, stream));
  const int64_t errs_cap = (cfg->record_errors && trace && trace->errors) ? trace->errors_cap : 0;
  double* d_errs = nullptr;
  if (errs_cap > 0) CUDA_TRY(arena.alloc(&d_errs, errs_cap));
  // emulated ranks: one exchange buffer per virtual rank, fresh per run
  char* vbuf = nullptr;
  if (L.vranks > 1 || !L.xbuf[0]) {
    const size_t xb = (xchg_bytes(L.P, L.nJ_cap, L.n_cap, G) + 255) & ~(size_t)255;
    CUDA_TRY(arena.alloc(&vbuf, xb * L.P));
    CUDA_TRY(cudaMemsetAsync(vbuf, 0, xb * L.P, stream));
    for (int q = 0; q < L.P; ++q) L.xbuf[q] = vbuf + q * xb;
  }

  SampleParams sp{};
  sp.key0 = cfg->philox_key[0];
  sp.key1 = cfg->philox_key[1];
  sp.draw_offset = cfg->draw_offset;
  sp.extended = extended;
  sp.n_row_blocks = (int32_t)s;
  sp.n_col_blocks = (int32_t)t;
  sp.row_ptr = d_row_ptr;
  sp.row_cum = d_row_cum;
  sp.row_total = cfg->row_total;
  sp.row_scale = d_row_scale;
  sp.col_ptr = d_col_ptr;
  sp.col_cum = d_col_cum;
  sp.col_total = cfg->col_total;
  sp.col_scale = d_col_scale;
  sp.picks = d_picks;

  StreamParams spar{};
  DenseParams& p = spar.d;
  p.A = ctx->A;
  p.lda = ctx->lda;
  p.m = (int32_t)ctx->m;
  p.n = (int32_t)ctx->n;
  p.b = b_dev;
  p.xs = xs_dev;
  p.x = x_dev;
  p.z = z_dev;
  p.upart = d_ws;
  p.rpart = d_ws + o_rpart;
  p.u = d_ws + o_u;
  p.r = d_ws + o_r;
  p.errpart = d_ws + o_err;
  p.errs = d_errs;
  p.errs_cap = errs_cap;
  p.plan = d_plan;
  p.ctl = d_ctl;
  p.extended = extended;
  p.stop_mode = cfg->stop_mode;
  p.tol = cfg->tol;
  p.stride = cfg->check_stride;
  p.max_iters = cfg->max_iters;
  p.res_scale = 1.0;
  p.record = errs_cap > 0;
  p.nonfinite_stop = cfg->nonfinite_stop;
  const char* prof_env = getenv("REBK_PROF");
  long long* d_prof = nullptr;
  const int Gtot = L.vranks * G;
  if (prof_env && prof_env[0] == '1') {
    CUDA_TRY(arena.alloc(&d_prof, (size_t)Gtot * 16));
    CUDA_TRY(cudaMemsetAsync(d_prof, 0, (size_t)Gtot * 16 * 8, stream));
  }
  p.prof = d_prof;
  spar.stages = stg.NS;
  spar.stage_doubles = stg.SD;
  spar.cw = stg.cw;
  spar.ch = stg.ch;
  spar.rw = stg.rw;
  spar.rh = stg.rh;
  spar.lc = stg.lc;
  spar.lr = stg.lr;
  spar.pad_nC = stg.pad_nC;
  spar.pad_nR = stg.pad_nR;
  spar.pad_nJ = stg.pad_nJ;
  spar.pad_nI = stg.pad_nI;
  spar.l2hint = env_int("REBK_STREAM_L2HINT", 1);
  spar.reverse = env_int("REBK_STREAM_REV", 1);
  spar.prefetch = env_int("REBK_STREAM_PF", 0);
  spar.pfence = env_int("REBK_STREAM_PFENCE", 0);
  spar.dbg = env_int("REBK_STREAM_DBG", 0);
  spar.order = env_int("REBK_STREAM_ORDER", 0);
  spar.tail = stream_tail(ctx, ctx->m, nJ_max, (int64_t)nI_loc * L.vranks, extended);
  double* d_zprev = nullptr;
  if (extended) CUDA_TRY(arena.alloc(&d_zprev, ctx->m));
  spar.zprev = d_zprev;
  RankXchg& X = spar.x;
  X.P = L.P;
  X.rank = L.rank;
  X.vranks = L.vranks;
  X.Gr = G;
  int64_t base = 0;
  for (int v = 0; v < L.vranks; ++v) {
    X.m[v] = (int32_t)L.rows[v];
    X.row_base[v] = (int32_t)base;
    base += L.rows[v];
  }
  X.x_stride = ctx->n;
  X.ws_stride = ws_stride;
  X.ranges = d_ranges;
  X.n_row_blocks = (int32_t)s;
  X.nJ_cap = (int32_t)L.nJ_cap;
  X.n_cap = L.n_cap;
  X.seq_base = L.seq_base;
  for (int q = 0; q < L.P; ++q) xchg_carve(L.xbuf[q], L.P, L.nJ_cap, L.n_cap, &X.inbox_u[q], &X.inbox_x[q], &X.flags[q]);

  cudaEvent_t ev0, ev1;
  CUDA_TRY(cudaEventCreate(&ev0));
  CUDA_TRY(cudaEventCreate(&ev1));
  cudaError_t err = cudaEventRecord(ev0, stream);
  int64_t k = 1;
  do {
    const int64_t count = std::min(chunk, cfg->max_iters - k + 1);
    if (err == cudaSuccess) err = launch_sample_plan(sp, k, count, d_plan, nullptr, stream);
    for (int v = 0; v < L.vranks && err == cudaSuccess; ++v)
      err = cudaMemsetAsync(&d_ctl[v].bar, 0, sizeof(unsigned long long), stream);
    p.k_begin = k;
    p.k_end = k + count - 1;
    if (err == cudaSuccess) err = launch_shard_stream(spar, tm_c, tm_r, stg.smem_bytes, stream);
    k += std::max<int64_t>(count, 1);
    if (err == cudaSuccess && k <= cfg->max_iters) {
      int32_t done = 0;
      err = cudaMemcpyAsync(&done, &d_ctl->done, sizeof done, cudaMemcpyDeviceToHost, stream);
      if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
      if (done) break;
    }
  } while (err == cudaSuccess && k <= cfg->max_iters);
  if (err == cudaSuccess) err = cudaEventRecord(ev1, stream);
  std::vector<Control> ctl(L.vranks);
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(ctl.data(), d_ctl, sizeof(Control) * L.vranks, cudaMemcpyDeviceToHost, stream);
  if (err == cudaSuccess && errs_cap > 0)
    err = cudaMemcpyAsync(trace->errors, d_errs, errs_cap * sizeof(double), cudaMemcpyDeviceToHost, stream);
  if (err == cudaSuccess) err = cudaStreamSynchronize(stream);
  float ms = 0.f;
  if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (err != cudaSuccess) return fail(REBK_ECUDA, "row-sharded REBK run failed: %s", cudaGetErrorString(err));
  for (int v = 0; v < L.vranks; ++v)
    if (ctl[v].fault)
      return fail(REBK_ECUDA, "row-sharded run: a cross-rank exchange timed out (a peer rank never arrived)");
  if (d_prof) {
    std::vector<long long> h((size_t)Gtot * 16);
    cudaMemcpy(h.data(), d_prof, h.size() * 8, cudaMemcpyDeviceToHost);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, ctx->device);
    const double it = (double)std::max<int64_t>(1, ctl[0].iters);
    fprintf(stderr, "[rebk prof] path=shard-stream P=%d vranks=%d Gr=%d iters=%lld loop=%.3f ms (%.3f us/iter); "
            "mark mean max\n", L.P, L.vranks, G, (long long)ctl[0].iters, ms, 1e3 * ms / it);
    print_prof(h, Gtot, Gtot, khz, it);
  }
  for (int v = 1; v < L.vranks; ++v)
    if (ctl[v].iters != ctl[0].iters || ctl[v].converged != ctl[0].converged)
      return fail(REBK_ECUDA, "row-sharded run: ranks stopped at different iterations (%lld vs %lld)",
                  (long long)ctl[v].iters, (long long)ctl[0].iters);
  if (trace) {
    trace->iters = ctl[0].iters;
    trace->converged = ctl[0].converged;
    trace->has_error = ctl[0].has_error;
    trace->final_error = ctl[0].final_error;
    trace->loop_ms = ms;
    trace->n_checks = ctl[0].n_checks;
    trace->grid_ctas = G;
    trace->kernel_path = 9;
    trace->nonfinite_at = ctl[0].nonfinite_at - 1;
  }
  // sequence numbers this solve used: the column sweep runs one step ahead of
  // the row sweep, so a run stopped at iteration K has exchanged u up to K + 1
  L.seq_base += (unsigned long long)ctl[0].iters + 2;
  if (ctl[0].nonfinite_at && cfg->nonfinite_stop)
    return fail(REBK_ENONFINITE, "non-finite error at the check of iteration %lld", (long long)(ctl[0].nonfinite_at - 1));
  return REBK_OK;
}

}  // namespace

namespace rebk {
int set_error_msg(int code, const char* msg) { return fail(code, "%s", msg); }
cudaError_t pool_malloc_bytes(void** p, size_t bytes) {
  cudaError_t e = cudaMallocAsync(p, bytes, cudaStreamPerThread);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamPerThread);
  return e;
}
void pool_free(void* p) {
  if (p) cudaFreeAsync(p, cudaStreamPerThread);
}
bool ctx_dense_view(const rebk_ctx* ctx, const double** A, int64_t* m, int64_t* n, int64_t* lda, int* device) {
  if (!ctx || ctx->kind != 0) return false;
  *A = ctx->A;
  *m = ctx->m;
  *n = ctx->n;
  *lda = ctx->lda;
  *device = ctx->device;
  return true;
}
}  // namespace rebk

extern "C" {

int rebk_abi_version(void) { return REBK_ABI_VERSION; }

int rebk_abi_struct_sizes(int64_t* cfg_size, int64_t* trace_size, int64_t* shard_args_size) {
  if (cfg_size) *cfg_size = (int64_t)sizeof(rebk_cfg);
  if (trace_size) *trace_size = (int64_t)sizeof(rebk_trace);
  if (shard_args_size) *shard_args_size = (int64_t)sizeof(rebk_shard_run_args);
  return REBK_OK;
}

const char* rebk_last_error(void) { return g_last_error.c_str(); }

int rebk_device_count(int* count) {
  if (!count) return fail(REBK_EINVAL, "null count");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(REBK_ENODEV, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = c;
  return REBK_OK;
}

static int ctx_common(rebk_ctx* c, int device) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(REBK_ENODEV, "no CUDA device available");
  if (device < 0 || device >= ndev) return fail(REBK_EINVAL, "device %d out of range", device);
  CUDA_TRY(cudaSetDevice(device));
  {
    // keep freed pool memory mapped (pool_malloc): see rebk_internal.h
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  CUDA_TRY(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  c->device = device;
  return REBK_OK;
}

int rebk_ctx_create_dense(const double* a_host, int64_t m, int64_t n, int64_t lda, int device,
                          rebk_ctx** out) {
  if (!out || !a_host) return fail(REBK_EINVAL, "null argument");
  if (m < 1 || n < 1) return fail(REBK_EINVAL, "matrix must be 2-D and nonempty");
  if (lda < n) return fail(REBK_EINVAL, "lda < n");
  rebk_ctx* c = new rebk_ctx{};
  int rc = ctx_common(c, device);
  if (rc) {
    delete c;
    return rc;
  }
  // store with an even leading dimension so every row is 16-byte aligned
  const int64_t ld = (n + 1) & ~(int64_t)1;
  double* dA = nullptr;
  cudaError_t e = pool_malloc(&dA, (size_t)m * ld);
  if (e != cudaSuccess) {
    delete c;
    return fail(REBK_ENOMEM, "cudaMalloc(A, %lld bytes): %s", (long long)(m * ld * 8), cudaGetErrorString(e));
  }
  if (ld != n) cudaMemset(dA, 0, (size_t)m * ld * sizeof(double));
  e = cudaMemcpy2D(dA, ld * sizeof(double), a_host, lda * sizeof(double), n * sizeof(double), m,
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(dA);
    delete c;
    return fail(REBK_ECUDA, "upload of A failed: %s", cudaGetErrorString(e));
  }
  c->m = m;
  c->n = n;
  c->lda = ld;
  c->A = dA;
  c->A_owned = dA;
  *out = c;
  return REBK_OK;
}

int rebk_ctx_create_dense_device(const double* a_dev, int64_t m, int64_t n, int64_t lda, int device,
                                 rebk_ctx** out) {
  if (!out || !a_dev) return fail(REBK_EINVAL, "null argument");
  if (m < 1 || n < 1) return fail(REBK_EINVAL, "matrix must be 2-D and nonempty");
  if (lda < n) return fail(REBK_EINVAL, "lda < n");
  rebk_ctx* c = new rebk_ctx{};
  int rc = ctx_common(c, device);
  if (rc) {
    delete c;
    return rc;
  }
  c->m = m;
  c->n = n;
  c->lda = lda;
  c->A = a_dev;
  c->A_owned = nullptr;
  *out = c;
  return REBK_OK;
}

int rebk_ctx_create_csr(const int64_t* indptr, const int32_t* indices, const double* data, int64_t m, int64_t n,
                        int64_t nnz, int device, rebk_ctx** out) {
  if (!out || !indptr || (nnz > 0 && (!indices || !data))) return fail(REBK_EINVAL, "null argument");
  if (m < 1 || n < 1) return fail(REBK_EINVAL, "matrix must be 2-D and nonempty");
  if (m > INT32_MAX || n > INT32_MAX) return fail(REBK_EINVAL, "matrix dimension exceeds 2^31");
  if (indptr[0] != 0 || indptr[m] != nnz) return fail(REBK_EINVAL, "indptr does not describe nnz entries");
  {
    // the reference Matrix's invariants (matrix.py:46-58), checked on up to
    // 16 host threads over row ranges; the first bad row in row order wins
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>({16, (int64_t)std::thread::hardware_concurrency(),
                                                               m / 4096 + 1}));
    std::vector<int64_t> bad_row(T, INT64_MAX);
    std::vector<int> bad_kind(T, 0);
    parallel_for_threads(T, [&](int th) {
      for (int64_t i = m * th / T; i < m * (th + 1) / T; ++i) {
        int kind = 0;
        if (indptr[i + 1] < indptr[i]) kind = 1;
        for (int64_t e = indptr[i]; !kind && e < indptr[i + 1]; ++e) {
          if (indices[e] < 0 || indices[e] >= n) kind = 2;
          else if (e > indptr[i] && indices[e] <= indices[e - 1]) kind = 3;
        }
        if (kind) {
          bad_row[th] = i;
          bad_kind[th] = kind;
          return;
        }
      }
    });
    for (int th = 0; th < T; ++th) {
      if (bad_kind[th] == 1) return fail(REBK_EINVAL, "indptr must be nondecreasing");
      if (bad_kind[th] == 2) return fail(REBK_EINVAL, "column index out of range");
      if (bad_kind[th] == 3) return fail(REBK_EINVAL, "column indices must be sorted and unique within a row");
    }
  }
  rebk_ctx* c = new rebk_ctx{};
  int rc = ctx_common(c, device);
  if (rc) {
    delete c;
    return rc;
  }
  c->kind = 1;
  c->m = m;
  c->n = n;
  c->lda = n;
  c->nnz = nnz;
  // upload the CSR (the caller's buffers; pinned ones copy at full PCIe
  // rate), then build the CSC twin on the device (rebk_csr_build.cu)
  cudaError_t e = pool_malloc(&c->csr_ptr, m + 1);
  if (!e) e = pool_malloc(&c->csr_col, nnz);
  if (!e) e = pool_malloc(&c->csr_val, nnz);
  if (!e) e = pool_malloc(&c->csc_ptr, n + 1);
  if (!e) e = pool_malloc(&c->csc_row, nnz);
  if (!e) e = pool_malloc(&c->csc_val, nnz);
  cudaStream_t st = nullptr;
  if (!e) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (!e) e = cudaMemcpyAsync(c->csr_ptr, indptr, sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, st);
  if (!e && nnz) e = cudaMemcpyAsync(c->csr_col, indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st);
  if (!e && nnz) e = cudaMemcpyAsync(c->csr_val, data, sizeof(double) * nnz, cudaMemcpyHostToDevice, st);
  if (!e) e = csr_to_csc_device(m, n, nnz, c->csr_ptr, c->csr_col, c->csr_val, c->csc_ptr, c->csc_row, c->csc_val, st);
  if (st) cudaStreamDestroy(st);
  if (e) {
    rebk_ctx_destroy(c);
    return fail(REBK_ENOMEM, "CSR upload / CSC twin failed: %s", cudaGetErrorString(e));
  }
  *out = c;
  return REBK_OK;
}

int rebk_ctx_create_dense_f32(const float* a_host, int64_t m, int64_t n, int64_t lda, int device, rebk_ctx** out) {
  if (!out || !a_host) return fail(REBK_EINVAL, "null argument");
  if (m < 1 || n < 1) return fail(REBK_EINVAL, "matrix must be 2-D and nonempty");
  if (lda < n) return fail(REBK_EINVAL, "lda < n");
  if (m > INT32_MAX || n > INT32_MAX) return fail(REBK_EINVAL, "matrix dimension exceeds 2^31");
  rebk_ctx* c = new rebk_ctx{};
  int rc = ctx_common(c, device);
  if (rc) {
    delete c;
    return rc;
  }
  float* dA = nullptr;
  cudaError_t e = pool_malloc(&dA, (size_t)m * n);
  if (e == cudaSuccess)
    e = cudaMemcpy2D(dA, n * sizeof(float), a_host, lda * sizeof(float), n * sizeof(float), m, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(dA);
    delete c;
    return fail(REBK_ENOMEM, "upload of fp32 A failed: %s", cudaGetErrorString(e));
  }
  c->kind = 2;
  c->m = m;
  c->n = n;
  c->lda = n;
  c->A32 = dA;
  *out = c;
  return REBK_OK;
}

int rebk_run_mrhs(rebk_ctx* ctx, const rebk_cfg* cfg, int64_t nrhs, const float* B, const float* X0, const float* Z0,
                  const float* Xstar, const double* tols, float* X_out, float* Z_out, int64_t* iters_out,
                  double* errs_out, rebk_trace* trace) {
  if (!ctx || !cfg || !B || !X_out || nrhs < 1) return fail(REBK_EINVAL, "null argument");
  if (ctx->kind != 2) return fail(REBK_EINVAL, "rebk_run_mrhs needs an fp32 context (rebk_ctx_create_dense_f32)");
  if (cfg->algorithm < 0 || cfg->algorithm > 3) return fail(REBK_EINVAL, "unknown algorithm %d", cfg->algorithm);
  if (cfg->stop_mode == REBK_STOP_RESIDUAL_PROXY)
    return fail(REBK_EINVAL, "multi-RHS runs support oracle_error and max_iters_only stopping");
  if (cfg->stop_mode == REBK_STOP_ORACLE_ERROR && !Xstar)
    return fail(REBK_EINVAL, "oracle_error stopping needs a problem with x_star");
  if (cfg->check_stride < 1) return fail(REBK_EINVAL, "check_stride must be at least 1");
  if (cfg->max_iters < 0) return fail(REBK_EINVAL, "max_iters must be nonnegative");
  const bool extended = cfg->algorithm == REBK_ALGO_REBK || cfg->algorithm == REBK_ALGO_REK;
  int rc = check_partition("row", cfg->n_row_blocks, cfg->row_ptr, cfg->row_cum, cfg->row_scale, ctx->m);
  if (rc) return rc;
  if (extended) {
    rc = check_partition("col", cfg->n_col_blocks, cfg->col_ptr, cfg->col_cum, cfg->col_scale, ctx->n);
    if (rc) return rc;
  }
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t stream;
  CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  const int64_t m = ctx->m, n = ctx->n, R = nrhs;
  rc = REBK_OK;
  {
    DevArena arena;
    arena.stream = stream;
    float *dB, *dX, *dZ = nullptr, *dXs = nullptr;
    int64_t *d_row_ptr, *d_col_ptr = nullptr;
    double *d_row_cum, *d_row_scale, *d_col_cum = nullptr, *d_col_scale = nullptr;
    const int64_t s = cfg->n_row_blocks, t = extended ? cfg->n_col_blocks : 0;
    cudaError_t e = arena.alloc(&dB, m * R);
    if (!e) e = arena.alloc(&dX, n * R);
    if (!e && extended) e = arena.alloc(&dZ, m * R);
    if (!e && Xstar) e = arena.alloc(&dXs, n * R);
    if (!e) e = cudaMemcpyAsync(dB, B, sizeof(float) * m * R, cudaMemcpyHostToDevice, stream);
    if (!e) e = X0 ? cudaMemcpyAsync(dX, X0, sizeof(float) * n * R, cudaMemcpyHostToDevice, stream)
                   : cudaMemsetAsync(dX, 0, sizeof(float) * n * R, stream);
    if (!e && extended) e = cudaMemcpyAsync(dZ, Z0 ? Z0 : B, sizeof(float) * m * R, cudaMemcpyHostToDevice, stream);
    if (!e && Xstar) e = cudaMemcpyAsync(dXs, Xstar, sizeof(float) * n * R, cudaMemcpyHostToDevice, stream);
    if (!e) e = arena.alloc(&d_row_ptr, s + 1);
    if (!e) e = arena.alloc(&d_row_cum, s);
    if (!e) e = arena.alloc(&d_row_scale, s);
    if (!e) e = cudaMemcpyAsync(d_row_ptr, cfg->row_ptr, (s + 1) * 8, cudaMemcpyHostToDevice, stream);
    if (!e) e = cudaMemcpyAsync(d_row_cum, cfg->row_cum, s * 8, cudaMemcpyHostToDevice, stream);
    if (!e) e = cudaMemcpyAsync(d_row_scale, cfg->row_scale, s * 8, cudaMemcpyHostToDevice, stream);
    if (!e && extended) {
      e = arena.alloc(&d_col_ptr, t + 1);
      if (!e) e = arena.alloc(&d_col_cum, t);
      if (!e) e = arena.alloc(&d_col_scale, t);
      if (!e) e = cudaMemcpyAsync(d_col_ptr, cfg->col_ptr, (t + 1) * 8, cudaMemcpyHostToDevice, stream);
      if (!e) e = cudaMemcpyAsync(d_col_cum, cfg->col_cum, t * 8, cudaMemcpyHostToDevice, stream);
      if (!e) e = cudaMemcpyAsync(d_col_scale, cfg->col_scale, t * 8, cudaMemcpyHostToDevice, stream);
    }
    if (e) {
      rc = fail(REBK_ECUDA, "multi-RHS upload failed: %s", cudaGetErrorString(e));
    } else {
      SampleParams sp{};
      sp.key0 = cfg->philox_key[0];
      sp.key1 = cfg->philox_key[1];
      sp.draw_offset = cfg->draw_offset;
      sp.extended = extended;
      sp.n_row_blocks = (int32_t)s;
      sp.n_col_blocks = (int32_t)t;
      sp.row_ptr = d_row_ptr;
      sp.row_cum = d_row_cum;
      sp.row_total = cfg->row_total;
      sp.row_scale = d_row_scale;
      sp.col_ptr = d_col_ptr;
      sp.col_cum = d_col_cum;
      sp.col_total = cfg->col_total;
      sp.col_scale = d_col_scale;
      // the tensor-core path reads column blocks as rows of Aᵀ (kind::tf32
      // operands must be K-major): one transposed copy per context
      const char* mm = getenv("REBK_MRHS_MATH");
      float* a32t = nullptr;
      int64_t ldat = 0;
      if ((!mm || !strcmp(mm, "tc")) && m % 4 == 0 && n % 4 == 0) {
        // built once per ctx under its mutex; published only after the
        // transpose finished, so a concurrent run never reads a partial copy
        std::lock_guard<std::mutex> lock(ctx->mu);
        if (!ctx->A32t) {
          float* t32 = nullptr;
          if (pool_malloc(&t32, (size_t)n * m) == cudaSuccess) {
            if (mrhs_transpose_a(ctx->A32, m, n, ctx->lda, t32, m, stream) == cudaSuccess &&
                cudaStreamSynchronize(stream) == cudaSuccess) {
              ctx->ldat = m;
              ctx->A32t = t32;
            } else {
              cudaGetLastError();
              cudaFree(t32);
            }
          } else {
            cudaGetLastError();
          }
        }
        a32t = ctx->A32t;
        ldat = ctx->ldat;
      }
      MrhsRun w{ctx->A32, m, n, ctx->lda, a32t, ldat, (int)R, dB, dX, dZ, dXs, cfg, tols, extended};
      double ms = 0.0;
      int64_t K = 0;
      int math = 0;
      char buf[512] = {0};
      std::vector<int64_t> it(R, -1);
      std::vector<double> er(R, 0.0);
      int r2 = run_mrhs(w, sp, nullptr, it.data(), er.data(), &ms, &K, buf, sizeof buf, stream, &math);
      if (r2) {
        rc = fail(REBK_ECUDA, "multi-RHS run failed: %s", buf);
      } else {
        bool all = cfg->stop_mode == REBK_STOP_ORACLE_ERROR;
        for (int64_t c = 0; c < R; ++c) {
          if (it[c] < 0) {
            all = false;
            it[c] = cfg->max_iters;
          }
        }
        if (iters_out) memcpy(iters_out, it.data(), sizeof(int64_t) * R);
        if (errs_out) memcpy(errs_out, er.data(), sizeof(double) * R);
        e = cudaMemcpyAsync(X_out, dX, sizeof(float) * n * R, cudaMemcpyDeviceToHost, stream);
        if (!e && Z_out && extended) e = cudaMemcpyAsync(Z_out, dZ, sizeof(float) * m * R, cudaMemcpyDeviceToHost, stream);
        if (!e) e = cudaStreamSynchronize(stream);
        if (e) rc = fail(REBK_ECUDA, "multi-RHS download failed: %s", cudaGetErrorString(e));
        if (trace) {
          trace->iters = K;
          trace->converged = all;
          trace->has_error = cfg->stop_mode == REBK_STOP_ORACLE_ERROR;
          trace->final_error = 0.0;
          for (int64_t c = 0; c < R; ++c) trace->final_error = std::max(trace->final_error, er[c]);
          trace->loop_ms = ms;
          trace->n_checks = 0;
          trace->grid_ctas = 0;
          trace->kernel_path = math == 6 ? 8 : (math == 4 ? 5 : 4);
          trace->nonfinite_at = -1;
          for (int64_t c = 0; c < R; ++c)
            if (!(er[c] - er[c] == 0.0)) trace->nonfinite_at = K;  // per-column errors at the stop: NaN/Inf
        }
      }
    }
  }
  cudaStreamSynchronize(stream);
  cudaStreamDestroy(stream);
  return rc;
}

static int shard_scratch(rebk_ctx* ctx, size_t len, double** out) {
  if (ctx->shard_scratch_len < len) {
    cudaFree(ctx->shard_scratch);
    ctx->shard_scratch = nullptr;
    ctx->shard_scratch_len = 0;
    CUDA_TRY(cudaMalloc(&ctx->shard_scratch, len * sizeof(double)));
    ctx->shard_scratch_len = len;
  }
  *out = ctx->shard_scratch;
  return REBK_OK;
}

int rebk_shard_colstep(rebk_ctx* ctx, int64_t c_lo, int64_t c_hi, const double* z_dev, double* u_dev, void* stream) {
  if (!ctx || ctx->kind != 0 || !z_dev || !u_dev || c_lo < 0 || c_hi > ctx->n || c_hi <= c_lo)
    return fail(REBK_EINVAL, "rebk_shard_colstep: bad argument");
  if (c_hi - c_lo > 512) return fail(REBK_EINVAL, "rebk_shard_colstep: column blocks up to 512 wide");
  CUDA_TRY(cudaSetDevice(ctx->device));
  double* scr = nullptr;
  int rc = shard_scratch(ctx, shard_colstep_scratch(ctx->m, c_hi - c_lo), &scr);
  if (rc) return rc;
  CUDA_TRY(shard_colstep(ctx->A, ctx->lda, ctx->m, c_lo, (int)(c_hi - c_lo), z_dev, u_dev, scr, (cudaStream_t)stream));
  return REBK_OK;
}

int rebk_shard_zupdate(rebk_ctx* ctx, int64_t c_lo, int64_t c_hi, double scale, const double* u_dev, double* z_dev,
                       void* stream) {
  if (!ctx || ctx->kind != 0 || !z_dev || !u_dev || c_lo < 0 || c_hi > ctx->n || c_hi <= c_lo)
    return fail(REBK_EINVAL, "rebk_shard_zupdate: bad argument");
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(shard_zupd(ctx->A, ctx->lda, ctx->m, c_lo, (int)(c_hi - c_lo), scale, u_dev, z_dev, (cudaStream_t)stream));
  return REBK_OK;
}

int rebk_shard_rowstep(rebk_ctx* ctx, const int64_t* rows_dev, int64_t nrows, const double* x_dev, const double* b_dev,
                       const double* z_dev, double* dx_dev, void* stream) {
  if (!ctx || ctx->kind != 0 || (nrows > 0 && !rows_dev) || !x_dev || !b_dev || !dx_dev || nrows < 0)
    return fail(REBK_EINVAL, "rebk_shard_rowstep: bad argument");
  CUDA_TRY(cudaSetDevice(ctx->device));
  double* scr = nullptr;
  int rc = shard_scratch(ctx, shard_rowstep_scratch(nrows, ctx->n), &scr);
  if (rc) return rc;
  CUDA_TRY(shard_rowstep(ctx->A, ctx->lda, ctx->n, rows_dev, nrows, x_dev, b_dev, z_dev, scr, dx_dev,
                         (cudaStream_t)stream));
  return REBK_OK;
}

int rebk_shard_xupdate(int64_t n, double scale, const double* dx_dev, double* x_dev, void* stream) {
  if (n < 1 || !dx_dev || !x_dev) return fail(REBK_EINVAL, "rebk_shard_xupdate: bad argument");
  CUDA_TRY(shard_xupd(n, scale, dx_dev, x_dev, (cudaStream_t)stream));
  return REBK_OK;
}

int rebk_shard_err2(int64_t n, const double* x_dev, const double* xs_dev, double* out_dev, void* stream) {
  if (n < 1 || !x_dev || !xs_dev || !out_dev) return fail(REBK_EINVAL, "rebk_shard_err2: bad argument");
  CUDA_TRY(shard_err(n, x_dev, xs_dev, out_dev, (cudaStream_t)stream));
  return REBK_OK;
}

/* ---- row-sharded multi-GPU path with the in-kernel exchange -------------- */
struct rebk_shard_xchg {
  int device = 0, P = 1, rank = 0, Gr = 0;
  int64_t nJ_cap = 0, n_cap = 0;
  char* buf = nullptr;  // this rank's exchange buffer (cudaMalloc: exportable by CUDA IPC)
  size_t bytes = 0, probe_off = 0;
  char* peer[kMaxRanks] = {};  // every rank's buffer mapped into this process (peer[rank] = buf)
  bool opened[kMaxRanks] = {};
  unsigned long long seq_base = 0;  // exchanges completed by earlier solves (identical on every rank)
  std::mutex mu;                    // one solve at a time per exchange object
};

int rebk_shard_grid_ctas(int device, int* grid_ctas) {
  if (!grid_ctas) return fail(REBK_EINVAL, "null argument");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) return fail(REBK_ENODEV, "no CUDA device");
  if (device < 0 || device >= n) return fail(REBK_EINVAL, "device %d out of range", device);
  int sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  *grid_ctas = sms;  // one CTA per SM (the kernel's shared-memory ring takes the SM)
  return REBK_OK;
}

int rebk_shard_xchg_create(int nranks, int rank, int64_t nJ_cap, int64_t n_cap, int grid_ctas, int device,
                           rebk_shard_xchg** out) {
  if (!out || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || nJ_cap < 1 || n_cap < 1 ||
      grid_ctas < 1)
    return fail(REBK_EINVAL, "rebk_shard_xchg_create: bad argument (at most %d ranks)", kMaxRanks);
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) return fail(REBK_ENODEV, "no CUDA device");
  CUDA_TRY(cudaSetDevice(device));
  rebk_shard_xchg* x = new rebk_shard_xchg();
  x->device = device;
  x->P = nranks;
  x->rank = rank;
  x->Gr = grid_ctas;
  x->nJ_cap = (nJ_cap + 1) & ~(int64_t)1;
  x->n_cap = (n_cap + 1) & ~(int64_t)1;
  // the protocol area, then kMaxRanks probe words (rebk_shard_xchg_probe)
  x->probe_off = (xchg_bytes(nranks, x->nJ_cap, x->n_cap, grid_ctas) + 255) & ~(size_t)255;
  x->bytes = x->probe_off + sizeof(unsigned long long) * kMaxRanks;
  cudaError_t e = cudaMalloc(&x->buf, x->bytes);
  if (e == cudaSuccess) e = cudaMemset(x->buf, 0, x->bytes);
  if (e != cudaSuccess) {
    cudaFree(x->buf);
    delete x;
    return fail(REBK_ENOMEM, "exchange buffer: %s", cudaGetErrorString(e));
  }
  x->peer[rank] = x->buf;
  *out = x;
  return REBK_OK;
}

int rebk_shard_xchg_ipc_handle(rebk_shard_xchg* x, unsigned char handle_out[64]) {
  if (!x || !handle_out) return fail(REBK_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(x->device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, x->buf));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle_out, &h, 64);
  return REBK_OK;
}

int rebk_shard_xchg_open_peers(rebk_shard_xchg* x, const unsigned char* handles) {
  if (!x || !handles) return fail(REBK_EINVAL, "null argument");
  CUDA_TRY(cudaSetDevice(x->device));
  for (int q = 0; q < x->P; ++q) {
    if (q == x->rank || x->opened[q]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * q, 64);
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    x->peer[q] = (char*)ptr;
    x->opened[q] = true;
  }
  return REBK_OK;
}

// Probe of the mapped peer buffers with the protocol's own instructions:
// phase 0 stores token * 16 + rank + 1 into probe word [rank] of EVERY rank's
// buffer (st.release.sys through the peer mapping); phase 1, called after a
// host-side barrier of the ranks, reads this rank's probe words
// (ld.acquire.sys) and counts the ranks whose word is missing.  Neither
// kernel waits on another rank's kernel.
struct ProbePeers {
  unsigned long long* w[kMaxRanks];
};
__global__ void shard_probe_post(ProbePeers pp, int P, int rank, unsigned long long token) {
  const int q = threadIdx.x;
  if (q < P)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pp.w[q] + rank), "l"(token * 16ull + (unsigned long long)rank + 1ull)
                 : "memory");
}
__global__ void shard_probe_check(const unsigned long long* mine, int P, unsigned long long token, int* missing) {
  const int q = threadIdx.x;
  if (q < P) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + q) : "memory");
    if (v != token * 16ull + (unsigned long long)q + 1ull) atomicAdd(missing, 1);
  }
}

int rebk_shard_xchg_probe(rebk_shard_xchg* x, int phase, uint64_t token, int* missing_out) {
  if (!x || (phase != 0 && phase != 1) || (phase == 1 && !missing_out)) return fail(REBK_EINVAL, "rebk_shard_xchg_probe: bad argument");
  for (int q = 0; q < x->P; ++q)
    if (!x->peer[q]) return fail(REBK_EINVAL, "rank %d's exchange buffer is not mapped (rebk_shard_xchg_open_peers)", q);
  CUDA_TRY(cudaSetDevice(x->device));
  std::lock_guard<std::mutex> lock(x->mu);
  if (phase == 0) {
    ProbePeers pp = {};
    for (int q = 0; q < x->P; ++q) pp.w[q] = (unsigned long long*)(x->peer[q] + x->probe_off);
    shard_probe_post<<<1, 32>>>(pp, x->P, x->rank, (unsigned long long)token);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return REBK_OK;
  }
  int* d_missing = nullptr;
  CUDA_TRY(cudaMalloc(&d_missing, sizeof(int)));
  cudaError_t e = cudaMemset(d_missing, 0, sizeof(int));
  if (e == cudaSuccess) {
    shard_probe_check<<<1, 32>>>((const unsigned long long*)(x->buf + x->probe_off), x->P, (unsigned long long)token, d_missing);
    e = cudaGetLastError();
  }
  int missing = -1;
  if (e == cudaSuccess) e = cudaMemcpy(&missing, d_missing, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d_missing);
  if (e != cudaSuccess) return fail(REBK_ECUDA, "rebk_shard_xchg_probe: %s", cudaGetErrorString(e));
  *missing_out = missing;
  return REBK_OK;
}

int rebk_shard_xchg_destroy(rebk_shard_xchg* x) {
  if (!x) return REBK_OK;
  cudaSetDevice(x->device);
  for (int q = 0; q < x->P; ++q)
    if (x->opened[q]) cudaIpcCloseMemHandle(x->peer[q]);
  cudaFree(x->buf);
  delete x;
  return REBK_OK;
}

int rebk_shard_run_device(rebk_ctx* ctx, rebk_shard_xchg* x, const rebk_cfg* cfg, const int64_t* local_ranges,
                          const double* b_dev, const double* x_star_dev, double* x_io_dev, double* z_io_dev,
                          void* stream, rebk_trace* trace) {
  if (!ctx || !x || !cfg || !local_ranges) return fail(REBK_EINVAL, "null argument");
  for (int q = 0; q < x->P; ++q)
    if (!x->peer[q]) return fail(REBK_EINVAL, "rank %d's exchange buffer is not mapped (rebk_shard_xchg_open_peers)", q);
  if (ctx->device != x->device) return fail(REBK_EINVAL, "ctx and exchange buffer live on different devices");
  std::lock_guard<std::mutex> lock(x->mu);
  ShardLaunch L;
  L.vranks = 1;
  L.P = x->P;
  L.rank = x->rank;
  L.Gr = x->Gr;
  const int64_t rows = ctx->m;
  L.rows = &rows;
  L.ranges = local_ranges;
  for (int q = 0; q < x->P; ++q) L.xbuf[q] = x->peer[q];
  L.nJ_cap = x->nJ_cap;
  L.n_cap = x->n_cap;
  L.seq_base = x->seq_base;
  const int rc = shard_stream_impl(ctx, cfg, L, b_dev, x_star_dev, x_io_dev, z_io_dev, (cudaStream_t)stream, trace);
  if (rc == REBK_OK || rc == REBK_ENONFINITE) x->seq_base = L.seq_base;
  return rc;
}

int rebk_shard_run_virtual(rebk_ctx* ctx, int vranks, const int64_t* rows_per_rank, const int64_t* local_ranges,
                           const rebk_cfg* cfg, const double* b_dev, const double* x_star_dev, double* x_io_dev,
                           double* z_io_dev, void* stream, rebk_trace* trace) {
  if (!ctx || !cfg || !rows_per_rank || !local_ranges) return fail(REBK_EINVAL, "null argument");
  if (vranks < 1 || vranks > kMaxRanks) return fail(REBK_EINVAL, "1..%d virtual ranks", kMaxRanks);
  ShardLaunch L;
  L.vranks = vranks;
  L.P = vranks;
  L.rank = 0;
  int G = cfg->grid_ctas > 0 ? cfg->grid_ctas : ctx->sm_count;
  L.Gr = std::max(1, G / vranks);
  L.rows = rows_per_rank;
  L.ranges = local_ranges;
  L.nJ_cap = std::max<int64_t>(2, (cfg->n_col_blocks > 0 && cfg->col_ptr) ? (max_block(cfg->n_col_blocks, cfg->col_ptr) + 1) & ~1 : 2);
  L.n_cap = (ctx->n + 1) & ~(int64_t)1;
  return shard_stream_impl(ctx, cfg, L, b_dev, x_star_dev, x_io_dev, z_io_dev, (cudaStream_t)stream, trace);
}

int rebk_ctx_destroy(rebk_ctx* ctx) {
  if (!ctx) return REBK_OK;
  if (ctx->shard_scratch) {
    cudaSetDevice(ctx->device);
    cudaFree(ctx->shard_scratch);
  }
  cudaSetDevice(ctx->device);
  // pool memory (pool_malloc): returned to the device pool, stays mapped
  for (void* p : {(void*)ctx->A32t, (void*)ctx->A32, (void*)ctx->A_owned, (void*)ctx->csr_ptr, (void*)ctx->csr_col,
                  (void*)ctx->csr_val, (void*)ctx->csc_ptr, (void*)ctx->csc_row, (void*)ctx->csc_val})
    pool_free(p);
  for (CsrSegPlan* sp : ctx->seg_cache) free_seg_plan(sp);
  cudaStreamSynchronize(cudaStreamPerThread);
  delete ctx;
  return REBK_OK;
}

int rebk_ctx_shape(const rebk_ctx* ctx, int64_t* m, int64_t* n) {
  if (!ctx) return fail(REBK_EINVAL, "null ctx");
  if (m) *m = ctx->m;
  if (n) *n = ctx->n;
  return REBK_OK;
}

int rebk_run_device(rebk_ctx* ctx, const rebk_cfg* cfg, const double* b_dev, const double* x_star_dev,
                    double* x_io_dev, double* z_io_dev, void* stream, rebk_trace* trace) {
  if (!ctx || !cfg) return fail(REBK_EINVAL, "null ctx/cfg");
  if (trace) trace->nonfinite_at = -1;
  return run_device_impl(ctx, cfg, b_dev, x_star_dev, x_io_dev, z_io_dev, (cudaStream_t)stream, trace);
}

int rebk_run(rebk_ctx* ctx, const rebk_cfg* cfg, const double* b, const double* x0, const double* z0,
             const double* x_star, double* x_out, double* z_out, rebk_trace* trace) {
  if (!ctx || !cfg || !b || !x_out) return fail(REBK_EINVAL, "null argument");
  if (trace) trace->nonfinite_at = -1;
  if (cfg->stop_mode == REBK_STOP_ORACLE_ERROR && !x_star)
    return fail(REBK_EINVAL, "oracle_error stopping needs a problem with x_star");
  const bool extended = cfg->algorithm == REBK_ALGO_REBK || cfg->algorithm == REBK_ALGO_REK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t stream;
  CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  const int64_t m = ctx->m, n = ctx->n;
  int rc = REBK_OK;
  {
    DevArena arena;
    arena.stream = stream;
    double *d_b, *d_x, *d_z = nullptr, *d_xs = nullptr;
    cudaError_t e = arena.alloc(&d_b, m);
    if (e == cudaSuccess) e = arena.alloc(&d_x, n);
    if (e == cudaSuccess && extended) e = arena.alloc(&d_z, m);
    if (e == cudaSuccess && x_star) e = arena.alloc(&d_xs, n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_b, b, m * 8, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
      e = x0 ? cudaMemcpyAsync(d_x, x0, n * 8, cudaMemcpyHostToDevice, stream)
             : cudaMemsetAsync(d_x, 0, n * 8, stream);
    if (e == cudaSuccess && extended)
      e = cudaMemcpyAsync(d_z, z0 ? z0 : b, m * 8, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && x_star) e = cudaMemcpyAsync(d_xs, x_star, n * 8, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) {
      rc = fail(REBK_ECUDA, "input upload failed: %s", cudaGetErrorString(e));
    } else {
      rc = run_device_impl(ctx, cfg, d_b, d_xs, d_x, d_z, stream, trace);
    }
    if (rc == REBK_OK || rc == REBK_ENONFINITE) {  // ENONFINITE: outputs hold the state of that check
      e = cudaMemcpyAsync(x_out, d_x, n * 8, cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess && z_out && extended)
        e = cudaMemcpyAsync(z_out, d_z, m * 8, cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) rc = fail(REBK_ECUDA, "output download failed: %s", cudaGetErrorString(e));
    }
  }
  cudaStreamSynchronize(stream);
  cudaStreamDestroy(stream);
  return rc;
}

int rebk_sample_sequence(const rebk_cfg* cfg, int64_t k0, int64_t count, int32_t* picks_out) {
  if (!cfg || !picks_out || k0 < 1 || count < 0) return fail(REBK_EINVAL, "bad argument");
  const bool extended = cfg->algorithm == REBK_ALGO_REBK || cfg->algorithm == REBK_ALGO_REK;
  const bool dsbgs = cfg->algorithm == REBK_ALGO_DSBGS;
  if (count == 0) return REBK_OK;
  if (dsbgs) {
    int rc = check_dsbgs(cfg);
    if (rc) return rc;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(REBK_ENODEV, "no CUDA device available");
  cudaStream_t stream;
  CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  int rc = REBK_OK;
  {
    DevArena arena;
    arena.stream = stream;
    SampleParams sp{};
    rebk_cfg c = *cfg;
    c.picks = nullptr;
    rc = upload_sampler(arena, &c, extended, extended || dsbgs, stream, &sp);
    int32_t* d_out = nullptr;
    cudaError_t e = cudaSuccess;
    if (!rc) e = arena.alloc(&d_out, 2 * count);
    if (!rc && !e) e = launch_sample_plan(sp, k0, count, nullptr, d_out, stream);
    if (!rc && !e) e = cudaMemcpyAsync(picks_out, d_out, 2 * count * sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
    if (!rc && !e) e = cudaStreamSynchronize(stream);
    if (!rc && e) rc = fail(REBK_ECUDA, "sampling failed: %s", cudaGetErrorString(e));
  }
  cudaStreamSynchronize(stream);
  cudaStreamDestroy(stream);
  return rc;
}

int rebk_block_frobenius_sq(rebk_ctx* ctx, int axis, int64_t nb, const int64_t* ptr, double* out) {
  if (!ctx || !ptr || !out || nb < 1 || (axis != 0 && axis != 1)) return fail(REBK_EINVAL, "bad argument");
  if (ctx->kind != 0 && ctx->kind != 2) return fail(REBK_EINVAL, "device block norms are implemented for dense matrices");
  const int64_t len = axis == 0 ? ctx->m : ctx->n;
  if (ptr[0] != 0 || ptr[nb] != len) return fail(REBK_EINVAL, "partition does not cover the axis");
  for (int64_t b = 0; b < nb; ++b)
    if (ptr[b + 1] < ptr[b]) return fail(REBK_EINVAL, "block pointers must be nondecreasing");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t stream;
  CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  int rc = REBK_OK;
  {
    DevArena arena;
    arena.stream = stream;
    int64_t* d_ptr;
    double* d_out;
    cudaError_t e = arena.alloc(&d_ptr, nb + 1);
    if (!e) e = arena.alloc(&d_out, nb);
    if (!e) e = cudaMemcpyAsync(d_ptr, ptr, (nb + 1) * 8, cudaMemcpyHostToDevice, stream);
    if (!e && ctx->kind == 2) {  // fp32 storage, fp64 accumulation
      double* d_part = nullptr;
      e = arena.alloc(&d_part, (size_t)(nb * block_norms_f32_scratch()));
      if (!e) e = launch_block_norms_f32(ctx->A32, ctx->lda, ctx->m, ctx->n, axis, nb, d_ptr, d_part, d_out, stream);
    } else if (!e) {
      e = launch_block_norms(ctx->A, ctx->lda, ctx->m, ctx->n, axis, nb, d_ptr, d_out, stream);
    }
    if (!e) e = cudaMemcpyAsync(out, d_out, nb * 8, cudaMemcpyDeviceToHost, stream);
    if (!e) e = cudaStreamSynchronize(stream);
    if (e) rc = fail(REBK_ECUDA, "block norms failed: %s", cudaGetErrorString(e));
  }
  cudaStreamSynchronize(stream);
  cudaStreamDestroy(stream);
  return rc;
}

int rebk_block_sigma1_sq(rebk_ctx* ctx, int axis, int64_t nb, const int64_t* ptr, int max_steps,
                         double* sigma1_sq_out, int32_t* steps_out) {
  if (!ctx || !ptr || !sigma1_sq_out || nb < 1 || (axis != 0 && axis != 1))
    return fail(REBK_EINVAL, "bad argument");
  if (ctx->kind != 0) return fail(REBK_EINVAL, "device block spectral norms are implemented for dense matrices");
  const int64_t len = axis == 0 ? ctx->m : ctx->n;
  if (ptr[0] != 0 || ptr[nb] != len) return fail(REBK_EINVAL, "partition does not cover the axis");
  for (int64_t b = 0; b < nb; ++b)
    if (ptr[b + 1] <= ptr[b]) return fail(REBK_EINVAL, "empty block in partition");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t stream;
  CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  const cudaError_t e = block_sigma1_sq(ctx->A, ctx->lda, ctx->m, ctx->n, axis, nb, ptr,
                                        max_steps > 0 ? max_steps : 300, sigma1_sq_out, steps_out, stream);
  cudaStreamDestroy(stream);
  if (e != cudaSuccess) return fail(REBK_ECUDA, "block spectral norms failed: %s", cudaGetErrorString(e));
  return REBK_OK;
}

int rebk_philox_key(const uint32_t* entropy_words, int64_t n_entropy_words, const uint32_t* spawn_words,
                    int64_t n_spawn_words, uint64_t key_out[2]) {
  if (!key_out || n_entropy_words < 0 || n_spawn_words < 0) return fail(REBK_EINVAL, "bad argument");
  std::vector<uint32_t> ent;
  if (n_entropy_words == 0)
    ent.push_back(0u);
  else
    ent.assign(entropy_words, entropy_words + n_entropy_words);
  if (n_spawn_words > 0) {
    while (ent.size() < 4) ent.push_back(0u);
    ent.insert(ent.end(), spawn_words, spawn_words + n_spawn_words);
  }
  seedseq_generate_u64x2(ent.data(), (int64_t)ent.size(), key_out);
  return REBK_OK;
}

int rebk_philox_uniforms_host(const uint64_t key[2], uint64_t first, int64_t count, double* out) {
  if (!key || !out || count < 0) return fail(REBK_EINVAL, "bad argument");
  for (int64_t q = 0; q < count; ++q) {
    const uint64_t d = first + (uint64_t)q;
    const u64x4 blk = philox_block(d >> 2, key[0], key[1]);
    out[q] = u64_to_unit_double(blk.v[d & 3]);
  }
  return REBK_OK;
}

int rebk_host_gather_col_blocks(const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t nb,
                                const int64_t* ptr, double* out, int nthreads) {
  if (!a || !ptr || !out || rows < 0 || nb < 1 || cols > lda || ptr[0] != 0 || ptr[nb] != cols)
    return fail(REBK_EINVAL, "rebk_host_gather_col_blocks: bad argument");
  for (int64_t k = 0; k < nb; ++k)
    if (ptr[k + 1] <= ptr[k]) return fail(REBK_EINVAL, "rebk_host_gather_col_blocks: empty or unordered block");
  if (rows == 0) return REBK_OK;
  // one sequential pass over A: row r's slice of block k lands at
  // out[rows*ptr[k] + r*w_k], i.e. every block as its own C-order array.
  // Threads own row slabs; the copy only moves bytes, so no result bit
  // depends on the thread count.
  int64_t nt = std::max<int64_t>(1, std::min<int64_t>(nthreads, (rows * cols) >> 16));
  nt = std::min<int64_t>(nt, rows);
  auto copy = [=](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) {
      const double* src = a + r * lda;
      for (int64_t k = 0; k < nb; ++k) {
        const int64_t w = ptr[k + 1] - ptr[k];
        memcpy(out + rows * ptr[k] + r * w, src + ptr[k], (size_t)w * sizeof(double));
      }
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(nt - 1);
  for (int64_t t = 1; t < nt; ++t) pool.emplace_back(copy, rows * t / nt, rows * (t + 1) / nt);
  copy(0, rows / nt);
  for (auto& th : pool) th.join();
  return REBK_OK;
}

}  // extern "C"

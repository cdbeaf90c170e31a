// rebk_internal.h — types shared by the sm_100a kernels and the C-ABI layer.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

struct rebk_cfg;
struct rebk_ctx;
namespace rebk {

constexpr int kThreads = 256;
// cluster shape of the clustered dense kernels (rebk_dense_fast.cu,
// rebk_dense_split.cu), fixed at compile time with __cluster_dims__
#ifndef REBK_CLUSTER_CS
#define REBK_CLUSTER_CS 8  // measured on C2: 6 -> 84.8 ms per solve, 8 -> 84.0 (profiles/r01_split_ncc_sweep.txt)
#endif
constexpr int kClusterCS = REBK_CLUSTER_CS;
constexpr int kWarps = kThreads / 32;
// dynamic shared memory we are willing to ask for (227 KB max per CTA on B200)
constexpr int kSmemBudget = 218 * 1024;

// One iteration's resolved picks (32 bytes): the column block [c_lo, c_hi)
// with its scale alpha/||A_{:,J}||_F^2 and the row block [r_lo, r_hi) with
// alpha/||A_{I,:}||_F^2 (solvers.py:151, :164).
struct Plan {
  int32_t c_lo, c_hi, r_lo, r_hi;
  double c_scale, r_scale;
  int32_t cb, rb;  // block indices (the sparse kernel indexes its per-block segment lists)
  int32_t pad0, pad1;
};

// Device-resident run control (one per rebk_run).
struct Control {
  unsigned long long bar;  // grid-barrier arrival counter (reset per launch)
  int32_t done;            // run finished (converged, or budget spent)
  int32_t converged;
  int64_t iters;
  double final_error;
  int64_t n_checks;
  int32_t has_error;
  int32_t fault;  // launch-shape mismatch detected on the device
  unsigned long long xseq;  // exchanges completed (fast path), carried across chunk launches
  unsigned long long xseq_row;  // split path: row-group exchanges
  int64_t nonfinite_at;  // 1 + first iteration whose stopping reduction was NaN/Inf (0: none)
};

// Split path: column-sweep group feeding the row-sweep group (rebk_dense_split.cu)
struct SplitShared {
  unsigned long long row_progress;  // last iteration whose z_I the row group has consumed
  unsigned long long stop;          // 0 running; K+1 = the run stopped with state K
};

// 16-byte {value, sequence} word of the fast path's cross-cluster exchange;
// written and read only through st_ll / poll_ll (rebk_device.cuh), which
// pack the sequence into both 8-byte halves so a torn access is detected
struct __align__(16) LLWord {
  unsigned long long half[2];  // {seq32 << 32 | lo32(v), seq32 << 32 | hi32(v)}
};

struct DenseParams {
  const double* A;
  int64_t lda;
  int32_t m, n;
  const double* b;
  const double* xs;  // x_star (oracle_error)
  double* x;
  double* z;
  // workspace (partials are stored transposed: part[e * G + g])
  double* upart;
  double* rpart;
  double* u;
  double* r;
  double* errpart;  // [G]
  double* res;      // [m] residual-proxy scratch
  double* errs;     // recorded errors
  int64_t errs_cap;
  const Plan* plan;  // plan[k - k_begin]
  int64_t k_begin, k_end;  // 1-based iterations handled by this launch
  Control* ctl;
  long long* prof;  // optional per-CTA phase cycle counters [G][16] (REBK_PROF=1)
  int32_t extended;   // REBK/REK: column sweep on z
  int32_t stop_mode;  // REBK_STOP_*
  double tol;
  int64_t stride;
  int64_t max_iters;
  double res_scale;
  int32_t record;
  int32_t nonfinite_stop;  // stop the run at a NaN/Inf error (rebk_cfg.nonfinite_stop)
  int32_t dsbgs;           // step_dsbgs: x update restricted to the plan's column block, no z
  // tile geometry (host-computed)
  int32_t nJ_max, nI_max;  // largest column / row block
  int32_t nR_max, nC_max;  // largest owned z-row / x-column slice
  int32_t ct_ld, rt_ld;    // leading dims of the staged tiles (doubles)
  int32_t stage_ct, stage_rt;  // 1 = tile staged in shared memory by TMA bulk copies
  int32_t ct_off, rt_off, vec_off;  // shared-memory carve-up (in doubles)
};

// fast path (rebk_dense_fast.cu): clustered exchanges, TMA 2D tiles
struct FastParams {
  DenseParams d;
  LLWord* cpart_u;  // [NC][stride_u] cluster partials of the u exchange (+ error entry)
  LLWord* cpart_r;  // [NC][stride_r] r partials, z_I, error entry
  int32_t stride_u, stride_r;
  int32_t ct_box_w, ct_box_h;  // TMA box of the column tile = its smem leading dim / rows
  int32_t rt_box_w, rt_box_h;
  int32_t pad_nC, pad_nR, pad_ne, pad_in, pad_cin;  // smem vector sizes (doubles, even)
  int32_t cluster_size;  // expected cluster size (checked on the device)
};

struct SplitParams {
  FastParams f;
  int32_t ncc;       // clusters [0, ncc) sweep columns (z), the rest sweep rows (x)
  int32_t ring;      // depth D of the z_I ring (column group may run D iterations ahead)
  int32_t hist;      // depth H of the z history (exact stop state), H >= D + 2
  int32_t zr_stride; // entries per ring slot (>= nI_max)
  LLWord* zring;     // [D][zr_stride] {z_{k,i}, seq = k}
  double* zhist;     // [H][m]
  SplitShared* sh;
  int32_t vec_off_c, vec_off_r;  // vector area base (doubles) of the column / row group
  int32_t xmode;                 // bit 0 / bit 1: column / row group exchanges gather all entries (no broadcast)
  int32_t pieces;                // TMA boxes per tile (1, or 2 row halves on separate mbarriers)
  unsigned long long* trace;     // REBK_TRACE: [trace_n][G][4] globaltimer stamps of the exchange stages
  int64_t trace_k0;
  int32_t trace_n;
};

// Streaming path for blocks too large for shared memory (rebk_dense_stream.cu):
// every pass streams TMA boxes through a ring of `stages` shared-memory stages.
constexpr int kStreamMaxStages = 8;
// Cross-rank exchange of the row-sharded streaming kernel:
// P ranks each hold interleaved rows of every row block; per iteration the
// |J|-length column product u and the n-length x update are summed over the
// ranks inside the persistent kernel.  Rank q's exchange buffer holds
//   inbox_u[2 slots][P][nJ_cap]  u partials of every rank (slot = k & 1)
//   inbox_x[2 slots][P][n_cap]   dx partials of every rank
//   flags[2 kinds][2 slots][P][Gr] u64 sequence numbers (kind 0: u, written
//                                  by CTA 0 of the sender; kind 1: x, written
//                                  by CTA g of the sender for its column slice)
// and every rank writes its partials into every rank's buffer (peer-mapped
// device memory over NVLink on a multi-GPU job; one allocation per virtual
// rank when `vranks` ranks are emulated in one launch on one GPU).  Every
// rank sums the P partials in rank order, so x stays bitwise replicated.
constexpr int kMaxRanks = 8;
struct RankXchg {
  int32_t P;        // ranks in the job (1: no exchange)
  int32_t rank;     // this process's rank (when vranks == 1)
  int32_t vranks;   // ranks emulated in this launch (1 on a real multi-GPU job)
  int32_t Gr;       // CTAs per rank (equal on every rank: x slices line up)
  int32_t m[kMaxRanks];         // local rows of each (virtual) rank
  int32_t row_base[kMaxRanks];  // first row of each virtual rank in the stacked A / b / z
  int64_t x_stride;   // doubles between virtual ranks' x arrays
  int64_t ws_stride;  // doubles between virtual ranks' workspaces (upart .. errpart)
  const int64_t* ranges;  // [vranks][n_row_blocks][2] local row range of each row block
  int32_t n_row_blocks;
  int32_t nJ_cap;
  int64_t n_cap;
  unsigned long long seq_base;  // per-solve epoch: sequence numbers are seq_base + k
  double* inbox_u[kMaxRanks];
  double* inbox_x[kMaxRanks];
  unsigned long long* flags[kMaxRanks];
};

struct StreamParams {
  DenseParams d;
  RankXchg x;  // row-sharded kernel only
  int32_t stages, stage_doubles;  // ring geometry (stage_doubles % 16 == 0)
  int32_t cw, ch;                 // column-block box: cw columns x ch rows
  int32_t rw, rh;                 // row-block box: rw columns x rh rows
  int32_t lc, lr;                 // lanes per row in the row dots (ch * lc, rh * lr <= 512)
  int32_t pad_nC, pad_nR, pad_nJ, pad_nI;  // vector areas after the ring (doubles, even)
  int32_t l2hint;   // 1: L2 eviction-priority hints on the TMA loads (REBK_STREAM_L2HINT, default 1)
  int32_t reverse;  // 1: second passes walk their row chunks backwards (REBK_STREAM_REV, default 1)
  int32_t prefetch; // boxes of L2 prefetch ahead of the TMA loads (REBK_STREAM_PF)
  int32_t pfence;   // fence.proxy.async before every TMA issue (REBK_STREAM_PFENCE, default 0)
  double* zprev;    // [m] z before the latest column sweep (written when a stop can be decided in the loop)
  int32_t tail;     // C1 row chunks (from the end) loaded evict_last for C2's backward walk (REBK_STREAM_TAIL)
  int32_t order;    // pass order within a step (REBK_STREAM_ORDER): 0 = C1 R1 | R2 C2, 1 = R1 C1 | C2 R2
  int32_t dbg;      // REBK_STREAM_DBG experiments (1: a third grid barrier at the end of every step)
};

// Sparse (CSR + CSC twin) persistent kernel (rebk_csr.cu).
struct CsrParams {
  int32_t m, n;
  const int64_t* csr_ptr;  // [m+1]
  const int32_t* csr_col;  // [nnz]
  const double* csr_val;
  const int64_t* csc_ptr;  // [n+1]
  const int32_t* csc_row;
  const double* csc_val;
  // per column block J: the block's rows with nonzeros (sorted), each with a
  // [ptr, ptr+1) range into compact copies of its entries (column order)
  const int64_t* cseg_off;  // [t+1]
  const int32_t* cseg_row;
  const int64_t* cseg_ptr;  // [nseg+1] into cval / ccol
  const double* cval;
  const int32_t* ccol;      // column - c_lo
  const int64_t* cseg_cta;  // [t][G+1] first segment of each CTA's z-row slice
  // per row block I: the block's columns with nonzeros (sorted), each with a
  // range into compact copies of its entries (row order)
  const int64_t* rseg_off;  // [s+1]
  const int32_t* rseg_col;
  const int64_t* rseg_ptr;
  const double* rval;
  const int32_t* rrow;      // row - r_lo
  const int64_t* rseg_cta;  // [s][G+1] first segment of each CTA's x-column slice
  const double* b;
  const double* xs;
  double* x;
  double* z;
  double* u;        // [nJ_max] column-sweep coefficients (global)
  double* r;        // [nI_max]
  double* errpart;  // [G]
  double* res;      // [m] residual-proxy scratch
  double* errs;
  int64_t errs_cap;
  const Plan* plan;
  int64_t k_begin, k_end;
  Control* ctl;
  int32_t extended;
  int32_t stop_mode;
  double tol;
  int64_t stride;
  int64_t max_iters;
  double res_scale;
  int32_t record;
  int32_t nonfinite_stop;
  int32_t dsbgs;  // step_dsbgs: x update restricted to the plan's column block, no z
  int32_t su_cap, sr_cap;  // u / r staged in shared memory (capacities in doubles, even; 0 = gathered from L2)
  int32_t specialize;      // independent parts of a phase on disjoint warps of the CTA (REBK_CSR_SPEC, default 1)
  int32_t l2_prefetch;  // bulk L2 prefetch of the next phases' block data (REBK_CSR_PF, default 1)
  long long* prof;  // optional per-CTA phase cycle counters [G][16] (REBK_PROF=1)
};

// One stopping check's bookkeeping, done by a single leader thread: the
// recorded error list, RunTrace.final_error (solvers.py:444-474) and the
// NaN/Inf detection.  Returns whether the run stops here; every CTA evaluates
// check_stops() on the same err, so they all agree without communication.
__host__ __device__ inline bool check_stops(double err, double tol, int32_t nonfinite_stop) {
  const bool bad = !(err - err == 0.0);  // NaN or +-Inf
  return err <= tol || (bad && nonfinite_stop);
}
__device__ inline void record_check(Control* ctl, double* errs, int64_t errs_cap, int32_t record, double err,
                                    double tol, int32_t nonfinite_stop, int64_t k) {
  const int64_t nc = ctl->n_checks;
  if (record && nc < errs_cap) errs[nc] = err;
  ctl->n_checks = nc + 1;
  ctl->final_error = err;
  ctl->has_error = 1;
  if (!(err - err == 0.0) && ctl->nonfinite_at == 0) ctl->nonfinite_at = k + 1;
  if (check_stops(err, tol, nonfinite_stop)) {
    ctl->converged = err <= tol;
    ctl->iters = k;
    ctl->done = 1;
  }
}

struct SampleParams {
  uint64_t key0, key1;
  uint64_t draw_offset;
  int32_t extended;
  int32_t n_row_blocks, n_col_blocks;
  const int64_t* row_ptr;
  const double* row_cum;
  double row_total;
  const double* row_scale;
  const int64_t* col_ptr;
  const double* col_cum;
  double col_total;
  const double* col_scale;
  const int32_t* picks;  // optional scripted picks, indexed by (k-1)
  // DSBGS joint sampler (rebk_cfg.dsbgs_*; device copies), dsbgs != 0
  int32_t dsbgs;
  const int64_t* d_off;
  const double* d_cum;
  const double* d_total;
  const int32_t* d_alive;
  const double* d_scale;
};

// balanced split of [0, len) over G parts; boundaries rounded down to even
// so that staged row segments start 16-byte aligned
__host__ __device__ inline int32_t split_even(int64_t len, int32_t G, int32_t g) {
  if (g >= G) return (int32_t)len;
  int64_t p = (len * (int64_t)g) / G;
  return (int32_t)(p & ~(int64_t)1);
}
__host__ __device__ inline int32_t split_rows(int64_t len, int32_t G, int32_t g) {
  if (g >= G) return (int32_t)len;
  return (int32_t)((len * (int64_t)g) / G);
}

// launchers (rebk_dense.cu)
cudaError_t launch_sample_plan(const SampleParams& sp, int64_t k0, int64_t count, Plan* plan,
                               int32_t* picks_out, cudaStream_t stream);
cudaError_t launch_dense(const DenseParams& p, int G, size_t smem_bytes, cudaStream_t stream);
// residual_proxy check between chunks of the fast dense kernels (rebk_dense.cu)
cudaError_t launch_residual_check(const double* A, int64_t lda, int m, int n, const double* x, const double* b,
                                  const double* z, double* res, double* part, double* colsq, double scale,
                                  double tol, int32_t nonfinite_stop, int32_t record, double* errs, int64_t errs_cap,
                                  int64_t k, Control* ctl, cudaStream_t st);
size_t residual_check_part_len(int m, int n);
cudaError_t dense_kernel_occupancy(size_t smem_bytes, int* blocks_per_sm);
cudaError_t launch_dense_fast(const FastParams& fp, const CUtensorMap& tm_ct, const CUtensorMap& tm_rt, int G,
                              int cluster_size, size_t smem_bytes, cudaStream_t stream);
cudaError_t fast_max_clusters(int cluster_size, size_t smem_bytes, int* clusters);
cudaError_t split_max_clusters(int cluster_size, size_t smem_bytes, int* clusters);
cudaError_t launch_dense_split(const SplitParams& sp, const CUtensorMap& tm_ct, const CUtensorMap& tm_rt, int G,
                               int cluster_size, size_t smem_bytes, cudaStream_t stream);
cudaError_t launch_dense_stream(const StreamParams& sp, const CUtensorMap& tm_c, const CUtensorMap& tm_r, int G,
                                size_t smem_bytes, cudaStream_t stream);
cudaError_t stream_kernel_occupancy(size_t smem_bytes, int* blocks_per_sm);
cudaError_t launch_shard_stream(const StreamParams& sp, const CUtensorMap& tm_c, const CUtensorMap& tm_r,
                                size_t smem_bytes, cudaStream_t stream);
cudaError_t launch_csr(const CsrParams& p, int G, cudaStream_t stream);
// Device memory that outlives one call (context arrays, cached plans): taken
// from the device's default memory pool, whose release threshold is raised
// when the first context is created, so a context created and destroyed per
// solve reuses mapped memory instead of paying cudaMalloc/cudaFree each time
cudaError_t pool_malloc_bytes(void** p, size_t bytes);
void pool_free(void* p);
template <class T>
inline cudaError_t pool_malloc(T** p, size_t count) {
  return pool_malloc_bytes(reinterpret_cast<void**>(p), (count > 0 ? count : 1) * sizeof(T));
}
// rebk_csr_build.cu: the sparse context's derived arrays built on the device
struct DevSegLists {
  int64_t nseg = 0;
  int64_t *off = nullptr, *ptr = nullptr, *cta = nullptr;
  int32_t *major_id = nullptr, *minor_local = nullptr;
  double* val = nullptr;
};
cudaError_t csr_to_csc_device(int64_t m, int64_t n, int64_t nnz, const int64_t* csr_ptr, const int32_t* csr_col,
                              const double* csr_val, int64_t* csc_ptr, int32_t* csc_row, double* csc_val,
                              cudaStream_t st);
cudaError_t seg_lists_device(int64_t nmajor, const int64_t* mptr, const int32_t* minor, const double* vals,
                             int64_t nnz, int64_t nminor, int64_t nb, const int64_t* bptr_host, int G, DevSegLists* out,
                             cudaStream_t st);
cudaError_t csr_kernel_occupancy(size_t smem_bytes, int* blocks_per_sm);
constexpr size_t kCsrStageBytesMax = 160 * 1024;  // shared memory the CSR kernel may use for the staged u and r
struct MrhsRun {
  const float* A;
  int64_t m, n, lda;
  const float* At;  // transposed copy (n x ldat) for the tensor-core path, or null
  int64_t ldat;
  int R;
  float *B, *X, *Z, *Xs;  // device, row-major (rows x R)
  const struct rebk_cfg* cfg;
  const double* tols;  // host [R]
  bool extended;
};
int run_mrhs(const MrhsRun& w, const SampleParams& sp_template, const SampleParams* unused, int64_t* iters_out,
             double* errs_out, double* loop_ms, int64_t* k_final, char* errbuf, size_t errlen, cudaStream_t stream,
             int* math_used);
// tensor-core (tcgen05, 3xTF32) multi-RHS path (rebk_mrhs_tc.cu)
bool mrhs_tc_supported(int64_t m, int64_t n, int R, int nJmax, int nImax);
cudaError_t mrhs_transpose_a(const float* A, int64_t m, int64_t n, int64_t lda, float* At, int64_t ldat,
                             cudaStream_t st);
int run_mrhs_tc(const MrhsRun& w, const SampleParams& sp_template, int64_t* iters_out, double* errs_out,
                double* loop_ms, int64_t* k_final, char* errbuf, size_t errlen, cudaStream_t stream);
// row-sharded multi-GPU pieces (rebk_shard.cu)
cudaError_t shard_colstep(const double* A, int64_t lda, int64_t m, int64_t c_lo, int nJ, const double* z, double* u,
                          double* scratch, cudaStream_t st);
cudaError_t shard_zupd(const double* A, int64_t lda, int64_t m, int64_t c_lo, int nJ, double s, const double* u,
                       double* z, cudaStream_t st);
cudaError_t shard_rowstep(const double* A, int64_t lda, int64_t n, const int64_t* rows, int64_t nrows, const double* x,
                          const double* b, const double* z, double* r_scratch, double* dx, cudaStream_t st);
// rebk_api.cu helpers for the other C-ABI files
int set_error_msg(int code, const char* msg);
bool ctx_dense_view(const rebk_ctx* ctx, const double** A, int64_t* m, int64_t* n, int64_t* lda, int* device);
size_t shard_colstep_scratch(int64_t m, int64_t nJ);
size_t shard_rowstep_scratch(int64_t nrows, int64_t n);
cudaError_t shard_xupd(int64_t n, double s, const double* dx, double* x, cudaStream_t st);
cudaError_t shard_err(int64_t n, const double* x, const double* xs, double* out, cudaStream_t st);
cudaError_t launch_block_norms(const double* A, int64_t lda, int64_t m, int64_t n, int axis,
                               int64_t nb, const int64_t* ptr_dev, double* out_dev,
                               cudaStream_t stream);
int64_t block_norms_f32_scratch();
cudaError_t launch_block_norms_f32(const float* A, int64_t lda, int64_t m, int64_t n, int axis, int64_t nb,
                                   const int64_t* ptr_dev, double* part_dev, double* out_dev, cudaStream_t stream);
// rebk_beta.cu: sigma_1(B_b)^2 of every block of a contiguous partition
cudaError_t block_sigma1_sq(const double* A, int64_t lda, int64_t m, int64_t n, int axis, int64_t nb,
                            const int64_t* h_ptr, int kmax, double* theta_out, int32_t* steps_out,
                            cudaStream_t stream);

}  // namespace rebk

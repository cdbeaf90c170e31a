/*
 * rebk.h — C ABI of librebk.so, the B200 (sm_100a) backend for the randomized
 * extended (average) block Kaczmarz iteration of arXiv 2001.04179.
 *
 * The reference (`kaczmarz`, pure Python, /root/reference/pkg) has no FFI; its
 * boundary for this path is Python-level:
 *   run(problem, config) -> RunTrace              solvers.py:425-474
 *   prepare(problem, config) -> SolverContext     solvers.py:271-273
 *   SolverContext.initial_state / .step           solvers.py:231-249, :267-268
 *   _STEPPERS[algo](state, ctx)                    solvers.py:384-392 (plugin point)
 * Each entry point below replaces one piece of that boundary; the citation on
 * each declaration names the reference code it stands in for.  Plain pointers
 * and sizes only: no torch / numpy types cross this ABI.
 *
 * Conventions
 *  - Every function returns 0 on success or a negative REBK_E* code; the
 *    message is kept per thread and read with rebk_last_error().
 *  - Dense A is row-major fp64 (m x n, leading dimension lda >= n), exactly
 *    the reference Matrix layout (matrix.py:37-44).
 *  - Row/column partitions are CONTIGUOUS blocks given by block pointers
 *    ptr[0]=0 < ptr[1] < ... < ptr[nb]=axis_len (sampling.py:107-112).  The
 *    host layer permutes A once for non-contiguous partitions.
 *  - The per-block sampling arrays (cumulative weights, total, alpha/w scales)
 *    are inputs, computed on the host exactly as the reference computes them
 *    (sampling.py:122-132, solvers.py:151/:164), so the device reproduces the
 *    reference block-index sequence bit for bit.
 *  - A rebk_ctx is immutable after creation ("Matrices are
 *    immutable"); concurrent rebk_run / rebk_run_device / rebk_run_mrhs
 *    calls on one ctx from different host threads are allowed (SPEC.md:390:
 *    distinct runs may execute concurrently): every run owns its workspace
 *    and stream, and the ctx's lazily built caches (sparse segment lists,
 *    the fp32 transposed copy) are built under the ctx's mutex and published
 *    only after their device copies completed.  Persistent kernels are
 *    launched cooperatively only, so two runs sharing a GPU serialise
 *    instead of deadlocking.  The rebk_shard_* pieces are the exception
 *    (documented below).
 */
#ifndef REBK_H
#define REBK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define REBK_ABI_VERSION 2

/* error codes */
#define REBK_OK 0
#define REBK_EINVAL -1     /* bad argument / dimension (reference: ValueError) */
#define REBK_ECUDA -2      /* CUDA runtime failure */
#define REBK_ENOMEM -3     /* device allocation failed */
#define REBK_ENODEV -4     /* no CUDA device */
#define REBK_ENONFINITE -5 /* NaN/Inf met in the stopping reduction */

/* algorithms served by the device kernel (solvers.py:39, :306-342) */
#define REBK_ALGO_REBK 0 /* step_rebk  solvers.py:324-337 */
#define REBK_ALGO_REK 1  /* step_rek   solvers.py:340-342 (singleton rebk) */
#define REBK_ALGO_RABK 2 /* step_rabk  solvers.py:315-321 (row sweep only) */
#define REBK_ALGO_RK 3   /* step_rk    solvers.py:306-312 (singleton rabk) */
#define REBK_ALGO_DSBGS 4 /* step_dsbgs solvers.py:371-381 (joint block sampler, dense A) */

/* stopping modes (solvers.py:50-70, :398-422) */
#define REBK_STOP_ORACLE_ERROR 0
#define REBK_STOP_RESIDUAL_PROXY 1
#define REBK_STOP_MAX_ITERS_ONLY 2

typedef struct rebk_ctx rebk_ctx;

/* One run's configuration: SolverConfig (solvers.py:73-85) with every
 * host-resolved quantity the device needs. */
typedef struct rebk_cfg {
  int32_t algorithm;     /* REBK_ALGO_* */
  int32_t stop_mode;     /* REBK_STOP_* */
  double tol;            /* StoppingRule.tol (absolute, solvers.py:61) */
  int64_t check_stride;  /* StoppingRule.check_stride */
  int64_t max_iters;     /* SolverConfig.max_iters */
  uint64_t philox_key[2];/* SeedSequence(seed).generate_state(2, u64) (sampling.py:36-37) */
  uint64_t draw_offset;  /* index of the first uniform this run consumes (0 for run()) */
  /* row partition (always present) */
  int64_t n_row_blocks;
  const int64_t* row_ptr;   /* [n_row_blocks+1] */
  const double* row_cum;    /* [n_row_blocks]  np.cumsum(weights) */
  double row_total;         /* cumulative[-1] */
  const double* row_scale;  /* [n_row_blocks]  alpha / w */
  /* column partition (REBK/REK only; 0/NULL for RABK/RK) */
  int64_t n_col_blocks;
  const int64_t* col_ptr;
  const double* col_cum;
  double col_total;
  const double* col_scale;
  /* optional explicit picks: [2*max_iters] int32 (col, row) per iteration,
   * used instead of the Philox stream (ScriptedRng in the reference tests,
   * test_solvers.py:23-31).  NULL = sample on device. */
  const int32_t* picks;
  int32_t record_errors;    /* SolverConfig.record_errors */
  int32_t grid_ctas;        /* 0 = automatic */
  double residual_scale;    /* sqrt(||A||_F^2) * ||b|| (solvers.py:411-413) */
  /* NaN/Inf in a stopping reduction: 0 = keep iterating like the reference
   * (run() has no finiteness check; the error stays NaN until max_iters,
   * solvers.py:444-474) and report it in rebk_trace.nonfinite_at; 1 = stop
   * at that check and return REBK_ENONFINITE (outputs hold that state). */
  int32_t nonfinite_stop;
  int32_t reserved0;
  /* REBK_ALGO_DSBGS only (solvers.py:204-229, _build_dsbgs_tables): the
   * joint law P(i, j) ~ ||A[I_i, J_j]||_F^2 as the column sampler (col_cum /
   * col_total above) times, per column block j, a conditional sampler over
   * the row blocks with a nonzero submatrix: entries [dsbgs_off[j],
   * dsbgs_off[j+1]) of dsbgs_cum (np.cumsum of those weights) and
   * dsbgs_alive (their row-block indices), total dsbgs_total[j];
   * dsbgs_scale[i * n_col_blocks + j] = alpha / ||A[I_i, J_j]||_F^2. */
  const int64_t* dsbgs_off;
  const double* dsbgs_cum;
  const double* dsbgs_total;
  const int32_t* dsbgs_alive;
  const double* dsbgs_scale;
} rebk_cfg;

/* RunTrace (solvers.py:96-112). errors is caller-allocated (capacity
 * errors_cap); checkpoints follow from (n_checks, check_stride, iters). */
typedef struct rebk_trace {
  int64_t iters;
  int32_t converged;
  int32_t has_error;        /* 0 when stop_mode == MAX_ITERS_ONLY */
  double final_error;
  double loop_ms;           /* device time of the iteration loop (CUDA events) */
  double* errors;
  int64_t errors_cap;
  int64_t n_checks;
  int32_t grid_ctas;        /* CTAs the persistent kernel used */
  int32_t kernel_path;      /* 0 dense general, 1 dense clustered, 2 same (cooperative), 3 sparse, 4/5 multi-RHS (5: BF16x9 tensor cores), 6 dense split column/row groups, 7 dense streaming (blocks larger than shared memory), 8 multi-RHS on hand-written tcgen05 3xTF32 kernels, 9 row-sharded streaming kernel with the in-kernel cross-rank exchange */
  int64_t nonfinite_at;     /* first check (iteration k) whose error was NaN/Inf; -1 if none */
} rebk_trace;

/* ---- library / device ---------------------------------------------------- */
int rebk_abi_version(void);
/* sizeof(rebk_cfg), sizeof(rebk_trace), sizeof(rebk_shard_run_args) as this
 * library was compiled (bindings check their struct mirrors against it) */
int rebk_abi_struct_sizes(int64_t* cfg_size, int64_t* trace_size, int64_t* shard_args_size);
const char* rebk_last_error(void);
int rebk_device_count(int* count);

/* ---- context: device copy of A (replaces Matrix dense storage,
 *      matrix.py:26-44, and the cached block views of
 *      SolverContext._materialize_blocks, solvers.py:115-120) --------------- */
int rebk_ctx_create_dense(const double* a_host, int64_t m, int64_t n, int64_t lda,
                          int device, rebk_ctx** out);
/* borrow an existing device array (caller keeps it alive; e.g. a torch tensor) */
int rebk_ctx_create_dense_device(const double* a_dev, int64_t m, int64_t n, int64_t lda,
                                 int device, rebk_ctx** out);
/* sparse A (replaces the CSR storage + CSC twin, matrix.py:46-58): CSR with
 * sorted unique column indices per row (the reference normalises to this,
 * matrix.py:226-231); the CSC twin is built inside.  The same rebk_run /
 * rebk_run_device entry points then run the sparse kernel. */
int rebk_ctx_create_csr(const int64_t* indptr, const int32_t* indices, const double* data, int64_t m,
                        int64_t n, int64_t nnz, int device, rebk_ctx** out);
int rebk_ctx_destroy(rebk_ctx* ctx);
int rebk_ctx_shape(const rebk_ctx* ctx, int64_t* m, int64_t* n);

/* ---- the hot path ---------------------------------------------------------
 * run(): solvers.py:425-474 with step_rebk / step_rek / step_rabk / step_rk.
 * Host buffers; copies in and out are part of the call.
 *   b [m] required; x0 [n] / z0 [m] optional (NULL -> x0 = 0, z0 = b,
 *   solvers.py:231-249); x_star [n] required for ORACLE_ERROR;
 *   x_out [n] required; z_out [m] optional. */
int rebk_run(rebk_ctx* ctx, const rebk_cfg* cfg, const double* b, const double* x0,
             const double* z0, const double* x_star, double* x_out, double* z_out,
             rebk_trace* trace);

/* Same with DEVICE buffers on `stream` (cudaStream_t as void*); x_io / z_io
 * hold the start point on entry (z_io ignored for RABK/RK) and the final
 * iterates on return.  Synchronises the stream before returning. */
int rebk_run_device(rebk_ctx* ctx, const rebk_cfg* cfg, const double* b_dev,
                    const double* x_star_dev, double* x_io_dev, double* z_io_dev,
                    void* stream, rebk_trace* trace);

/* ---- multi-RHS fp32 (BASELINE config 5; no reference counterpart: the
 * reference takes one 1-D b, solvers.py:141-143).  A fp32 row-major; B, X,
 * Z row-major with nrhs columns; every RHS shares the block sequence of
 * cfg (so each column follows exactly the single-RHS REBK of
 * solvers.py:324-337).  Column c stops counting at its first check with
 * ||X_c - X*_c|| <= tols[c]; the run ends when all columns have crossed
 * (trace->iters = that iteration, iters_out[c] = column c's first crossing)
 * and returns the state at that iteration. */
int rebk_ctx_create_dense_f32(const float* a_host, int64_t m, int64_t n, int64_t lda, int device,
                              rebk_ctx** out);
int rebk_run_mrhs(rebk_ctx* ctx, const rebk_cfg* cfg, int64_t nrhs, const float* B, const float* X0,
                  const float* Z0, const float* Xstar, const double* tols, float* X_out, float* Z_out,
                  int64_t* iters_out, double* errs_out, rebk_trace* trace);

/* ---- row-sharded multi-GPU pieces (BASELINE config 3).  ctx
 * holds this rank's rows of A; all buffers are device buffers on `stream`.
 * Between colstep and zupdate the caller allreduces u (|J| doubles), between
 * rowstep and xupdate it allreduces dx (n doubles), on its communicator.
 * Together they are one step_rebk (solvers.py:324-337) on the sharded A.
 * Fixed-order reductions; the ctx's scratch makes these calls non-reentrant
 * per ctx. rebk_shard_colstep takes column blocks up to 512 wide. */
int rebk_shard_colstep(rebk_ctx* ctx, int64_t c_lo, int64_t c_hi, const double* z_dev, double* u_dev,
                       void* stream);
int rebk_shard_zupdate(rebk_ctx* ctx, int64_t c_lo, int64_t c_hi, double scale, const double* u_dev,
                       double* z_dev, void* stream);
int rebk_shard_rowstep(rebk_ctx* ctx, const int64_t* rows_dev, int64_t nrows, const double* x_dev,
                       const double* b_dev, const double* z_dev, double* dx_dev, void* stream);
int rebk_shard_xupdate(int64_t n, double scale, const double* dx_dev, double* x_dev, void* stream);
int rebk_shard_err2(int64_t n, const double* x_dev, const double* xs_dev, double* out_dev, void* stream);

/* ---- row-sharded multi-GPU solve over NCCL (rebk_nccl.cu) ---------------
 * NCCL is loaded with dlopen from libnccl_path (the libnccl.so.2 torch uses;
 * NULL/"" = the loader's default).  Rank 0 creates the unique id, the
 * caller distributes it (e.g. torch.distributed broadcast), every rank
 * creates its communicator.  rebk_shard_run then runs a whole solve of this
 * rank's shard — the iteration sequence of run_sharded in sharded.py,
 * replacing step_rebk/run (solvers.py:324-337, :425-474) — issuing the
 * per-rank kernels and the two allreduces per iteration on one stream and
 * reading the device-side stop checks once per `chunk` iterations (exact
 * crossing by replay from the chunk's snapshot). */
typedef struct rebk_shard_run_args {
  int64_t max_iters;
  int64_t stride;
  double tol;              /* absolute, on ||x - x*|| */
  int32_t chunk;
  int32_t extended;        /* 1: REBK (column sweep), 0: RABK */
  const int32_t* picks;    /* host [max_iters][2]: column block (or -1), row block */
  int64_t n_col_blocks;
  const int64_t* col_ptr;  /* host [n_col_blocks + 1] */
  const double* col_scale; /* host [n_col_blocks] */
  int64_t n_row_blocks;
  const int64_t* row_ptr;  /* host [n_row_blocks + 1] (global; for validation) */
  const double* row_scale; /* host [n_row_blocks] */
  const int64_t* local_ranges;   /* host [n_row_blocks][2]: this rank's local rows of each block */
  const int64_t* local_rows_dev; /* device [m_local]: 0, 1, ..., m_local - 1 */
  const double* b_dev;     /* device [m_local] */
  double* x_dev;           /* device [n], in/out (replicated) */
  double* z_dev;           /* device [m_local], in/out */
  const double* xs_dev;    /* device [n] */
  int64_t n_picks;         /* entries of picks (>= max_iters); every pick is range-checked */
} rebk_shard_run_args;
int rebk_nccl_get_unique_id(const char* libnccl_path, unsigned char id_out[128]);
int rebk_nccl_comm_create(const char* libnccl_path, const unsigned char id[128], int nranks, int rank,
                          int device, void** comm_out);
int rebk_nccl_comm_destroy(void* comm);
int rebk_shard_run(rebk_ctx* ctx, void* comm, const rebk_shard_run_args* args, int64_t* iters_out,
                   int32_t* converged_out, double* final_err_out);

/* ---- row-sharded multi-GPU solve with the exchange INSIDE the persistent
 * kernel (rebk_shard_stream_kernel).  Every rank holds the
 * interleaved rows of every row block (local row q of block b on rank
 * floor(q P / |I_b|)), z and b follow the rows, x is replicated.  Per
 * iteration the |J| column-product partials and the n-length x-update
 * partials go straight from the kernel into every rank's exchange buffer
 * (peer memory over NVLink, mapped with CUDA IPC), each followed by a
 * release flag at system scope; every rank sums the P partials in rank
 * order, so x stays bitwise replicated and all ranks stop at the same check.
 * One launch per solve (per 2^20 iterations), no host work per iteration.
 * Replaces step_rebk/run (solvers.py:324-337, :425-474) on the sharded A.
 *
 *   rebk_shard_grid_ctas    CTAs per rank this device runs (all ranks must use the same value: take the min)
 *   rebk_shard_xchg_create  this rank's exchange buffer (nranks <= 8)
 *   rebk_shard_xchg_ipc_handle / _open_peers  export the buffer, map every peer's (handles: [nranks][64])
 *   rebk_shard_xchg_probe   checks the mapping with the protocol's own instructions: phase 0 stores a token word
 *                           into every rank's buffer (st.release.sys through the peer mapping); phase 1 (after a
 *                           host-side barrier of the ranks) counts the ranks whose word did not arrive here
 *   rebk_shard_run_device   one solve of this rank's shard; ctx = this rank's rows; cfg = the GLOBAL partitions
 *                           and sampler arrays (row_ptr of the whole matrix); local_ranges [n_row_blocks][2] =
 *                           this rank's rows of each block in local numbering; b_dev, z_io_dev local; x_io_dev,
 *                           x_star_dev replicated.  All ranks must call it the same number of times.
 *   rebk_shard_run_virtual  the same kernel with `vranks` ranks emulated in ONE cooperative launch on one GPU
 *                           (the ranks' rows stacked in ctx, rows_per_rank[vranks], local_ranges
 *                           [vranks][n_row_blocks][2], b/z stacked, x_io_dev [vranks][n]): tests the exchange
 *                           protocol where ranks that wait on each other must run at the same time.
 * A rank whose peer never arrives fails after 60 s (REBK_ECUDA) instead of hanging. */
typedef struct rebk_shard_xchg rebk_shard_xchg;
int rebk_shard_grid_ctas(int device, int* grid_ctas);
int rebk_shard_xchg_create(int nranks, int rank, int64_t nJ_cap, int64_t n_cap, int grid_ctas, int device,
                           rebk_shard_xchg** out);
int rebk_shard_xchg_ipc_handle(rebk_shard_xchg* x, unsigned char handle_out[64]);
int rebk_shard_xchg_open_peers(rebk_shard_xchg* x, const unsigned char* handles);
int rebk_shard_xchg_probe(rebk_shard_xchg* x, int phase, uint64_t token, int* missing_out);
int rebk_shard_xchg_destroy(rebk_shard_xchg* x);
int rebk_shard_run_device(rebk_ctx* ctx, rebk_shard_xchg* x, const rebk_cfg* cfg, const int64_t* local_ranges,
                          const double* b_dev, const double* x_star_dev, double* x_io_dev, double* z_io_dev,
                          void* stream, rebk_trace* trace);
int rebk_shard_run_virtual(rebk_ctx* ctx, int vranks, const int64_t* rows_per_rank, const int64_t* local_ranges,
                           const rebk_cfg* cfg, const double* b_dev, const double* x_star_dev, double* x_io_dev,
                           double* z_io_dev, void* stream, rebk_trace* trace);

/* ---- sampler (sampling.py:23-45 Rng, :137-145 WeightedSampler.sample) -----
 * Device sampling of the (col, row) block-index pairs of iterations
 * [k0, k0+count) (k is 1-based), written to picks_out[2*count] (host). */
int rebk_sample_sequence(const rebk_cfg* cfg, int64_t k0, int64_t count, int32_t* picks_out);

/* Device block Frobenius norms (matrix.py:170-189): out[nb] for contiguous
 * blocks ptr[nb+1] along axis 0 (rows) or 1 (columns).  Dense fp64 contexts
 * and fp32 contexts (rebk_ctx_create_dense_f32; squares accumulated in
 * fp64, i.e. the norms of the matrix's exact fp64 upcast). */
int rebk_block_frobenius_sq(rebk_ctx* ctx, int axis, int64_t nb, const int64_t* ptr,
                            double* out);

/* Device block spectral norms: sigma_1(B_b)^2 for the nb contiguous blocks
 * ptr[nb+1] along axis 0 (row blocks A[I,:]) or 1 (column blocks A[:,J]),
 * by Lanczos with full reorthogonalisation on the block's small Gram
 * operator (at most max_steps steps per block; <= 0 selects 300).  Replaces
 * the per-block Jacobi SVD of the reference's _block_beta (rates.py:76-90):
 * beta = max_b sigma1_sq_out[b] / ||B_b||_F^2.  steps_out (nullable)
 * receives the Lanczos steps each block took. */
int rebk_block_sigma1_sq(rebk_ctx* ctx, int axis, int64_t nb, const int64_t* ptr, int max_steps,
                         double* sigma1_sq_out, int32_t* steps_out);

/* ---- MatrixMarket -> CSR / dense host arrays (rebk_mmio.cpp) -------------
 * Native reader with the acceptance rules and error texts of the reference's
 * read_matrix_market (matrix_io.py:67-157): coordinate (real / integer /
 * pattern, general / symmetric) and array formats, duplicates summed,
 * symmetric storage mirrored, Python int()/float() token grammar, the
 * density threshold that decides dense vs CSR.  The output arrays (CSR with
 * sorted columns and no explicit zeros: the reference Matrix's normalised
 * form, ready for rebk_ctx_create_csr) are malloc'ed by the library and
 * released with rebk_mm_free.  On a parse error: REBK_EINVAL, the message
 * (without the "path:line: " prefix) in rebk_last_error, the 1-based line in
 * out->err_line.  Parses on up to nthreads host threads. */
typedef struct rebk_mm_matrix {
  int64_t rows, cols;
  int32_t dense;       /* 1: values = rows x cols row-major; 0: CSR */
  int32_t reserved;
  int64_t nnz;
  int64_t* indptr;     /* [rows + 1] (CSR) */
  int32_t* indices;    /* [nnz] */
  double* values;      /* [nnz] or [rows * cols] */
  int64_t err_line;
} rebk_mm_matrix;
int rebk_mm_read(const char* path, double dense_threshold, int nthreads, rebk_mm_matrix* out);
void rebk_mm_free(rebk_mm_matrix* m);

/* ---- host-side helpers (no GPU needed) ---------------------------------- */
/* numpy SeedSequence(entropy, spawn_key).generate_state(2, uint64): the
 * Philox key of Rng(seed, spawn_key) (sampling.py:33-37). entropy / spawn
 * words are the little-endian uint32 digits of each non-negative integer,
 * n_spawn_words[i] giving how many words spawn key i contributes. */
int rebk_philox_key(const uint32_t* entropy_words, int64_t n_entropy_words,
                    const uint32_t* spawn_words, int64_t n_spawn_words, uint64_t key_out[2]);
/* Uniform doubles draws [first, first+count) of Rng with this key
 * (Generator.random: (u64 >> 11) * 2^-53). */
int rebk_philox_uniforms_host(const uint64_t key[2], uint64_t first, int64_t count,
                              double* out);

/* Host-side helper for the sampler weights (matrix.py:170-189): one
 * sequential pass over a row-major host matrix (row stride lda) that writes
 * every column block ptr[k]..ptr[k+1] of a contiguous partition (ptr[0] = 0,
 * ptr[nb] = cols) as its own C-order array at out + rows*ptr[k] — the array
 * np.ravel(A[:, J]) builds — with up to nthreads host threads.  The weight
 * stays numpy's `flat @ flat` on that array, keeping the reference's bits. */
int rebk_host_gather_col_blocks(const double* a, int64_t rows, int64_t cols, int64_t lda, int64_t nb,
                                const int64_t* ptr, double* out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif /* REBK_H */

// rebk_dense_stream.cu — REBK for dense fp64 problems whose per-CTA block
// slices do not fit in shared memory (C3: 200000 x 10000, |J| = 500, |I| = 1000:
// a CTA's slice of the column block is ~1350 rows x 500 = 5.4 MB).
//
// Same iteration, ownership and reductions as rebk_dense.cu (step_rebk,
// solvers.py:324-337; partial sums stored transposed and summed in fixed
// order, so runs replay bit for bit).  What changes is the data movement:
// every pass over a block is a stream of TMA boxes through a ring of NS
// shared-memory stages, each on its own mbarrier.
//
// Schedule: in step_rebk the z sequence never depends on x, and the row sweep
// of iteration k needs only z_k[I_k].  So the two sweeps are software-
// pipelined one iteration apart and share their grid barriers: step s runs
//   X:  C1(s)  u partials          +  R1(s-1)  r partials     -> barrier, both sums
//   Y:  R2(s-1) x update           +  C2(s)    z update       (after a 2nd barrier)
// i.e. two grid barriers per iteration instead of four, and the row sweep's
// 160 MB ride in the column sweep's HBM stream instead of being two short
// phases of their own.  No barrier is needed between Y and the next X: C1 and
// R1 read only the CTA's own z rows / x columns, and the partial buffers they
// write were last read before the second barrier.  A stop decided for
// x_{s-2} (after the first barrier of step s) needs z_{s-2}, one column sweep
// back: C2 also stores the z it replaces (StreamParams.zprev).
// The chunk sequence of a whole run is known in advance (the block plan), so
// thread 0 keeps NS boxes in flight across phases and grid barriers: while a
// CTA waits at a barrier, the first boxes of the next pass are already
// landing.  Per iteration each CTA streams
//   C1  its rows of A[:, J]  (u partials, column sums)          HBM
//   C2  the same rows again  (z -= s_J A_J u, row dots)          HBM (800 MB does not stay in L2)
//   R1  A[I, its columns]    (r partials, row dots)              HBM
//   R2  the same again       (x -= s_I A_Iᵀ r, column sums)      L2  (80 MB, just read by R1)
// so the column block is read twice: the HBM floor is ~1.68 GB per C3
// iteration, 0.52 of the "blocks read once" algorithmic figure.
//
// The same body, instantiated with SH = true, is the row-sharded kernel of
// the multi-GPU path (rebk_shard_stream_kernel): each rank
// streams only its interleaved rows; after the local u sum the |J| values go
// to every rank's inbox (peer memory), and R2's column partials of x go the
// same way, CTA g to CTA g (the x column split is identical on every rank),
// each followed by a flag store with release semantics at system scope.
// Every rank then sums the P partials in rank order: no host round trip, no
// launch per iteration, x bitwise replicated so every rank stops at the
// same check.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rebk_device.cuh"
#include "rebk_internal.h"

namespace rebk {

constexpr int kStreamThreads = 512;
constexpr int kStreamWarps = kStreamThreads / 32;

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// a peer that never arrives (a rank that failed or was killed) must not hang
// the others forever: every cross-rank wait, and the rank-local barrier of the
// sharded kernel, gives up after this long and the run fails with an error
constexpr unsigned long long kXchgTimeoutNs = 60ull * 1000ull * 1000ull * 1000ull;

template <bool SH>
__device__ __forceinline__ void stream_body(const StreamParams& sp, const CUtensorMap& tm_c, const CUtensorMap& tm_r) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t sbar[kStreamMaxStages];
  __shared__ double s_bcast[2];

  const DenseParams& p = sp.d;
  const RankXchg& X = sp.x;
  // (virtual) rank of this CTA and its share of the launch
  const int vr = SH ? (int)blockIdx.x / X.Gr : 0;
  const int G = SH ? X.Gr : (int)gridDim.x;
  const int g = SH ? (int)blockIdx.x - vr * X.Gr : (int)blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int P = SH ? X.P : 1;
  // a single rank has nothing to exchange: the sharded kernel then takes the
  // single-GPU code paths (same bits, no flags or system-scope fences)
  const bool XCH = SH && P > 1;
  const int rank = SH ? (X.vranks > 1 ? vr : X.rank) : 0;
  const int m_loc = SH ? X.m[vr] : p.m;
  const int rbase = SH ? X.row_base[vr] : 0;
  const int64_t wso = SH ? (int64_t)vr * X.ws_stride : 0;
  const double* gb = p.b + rbase;
  double* gz = p.z ? p.z + rbase : nullptr;
  double* gzp = sp.zprev ? sp.zprev + rbase : nullptr;  // z before the latest column sweep (exact stop state)
  double* gx = p.x + (SH ? (int64_t)vr * X.x_stride : 0);
  double* upart = p.upart + wso;
  double* rpart = p.rpart + wso;
  double* gu = p.u + wso;
  double* gr = p.r + wso;
  double* errpart = p.errpart + wso;
  const int64_t* lrange = SH ? X.ranges + (int64_t)vr * 2 * X.n_row_blocks : nullptr;
  Control* ctl = p.ctl + vr;
  if (*((volatile int32_t*)&ctl->done)) return;

  const int zr0 = split_rows(m_loc, G, g), zr1 = split_rows(m_loc, G, g + 1);
  const int xq0 = split_even(p.n, G, g), xq1 = split_even(p.n, G, g + 1);
  const int nR = zr1 - zr0, nC = xq1 - xq0;
  const int NS = sp.stages, SD = sp.stage_doubles;
  const int cw = sp.cw, ch = sp.ch, rw = sp.rw, rh = sp.rh;

  double* s_x = sm + (size_t)NS * SD;
  double* s_xs = s_x + sp.pad_nC;
  double* s_z = s_xs + sp.pad_nC;
  double* s_u = s_z + sp.pad_nR;
  double* s_r = s_u + sp.pad_nJ;
  double* s_red = s_r + sp.pad_nI;  // 2 * kStreamThreads

  for (int c = tid; c < nC; c += kStreamThreads) {
    s_x[c] = __ldcg(gx + xq0 + c);
    s_xs[c] = p.xs ? __ldg(p.xs + xq0 + c) : 0.0;
  }
  if (p.extended)
    for (int r = tid; r < nR; r += kStreamThreads) s_z[r] = __ldcg(gz + zr0 + r);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&sbar[s], 1);
    fence_mbar_init();
    prefetch_tensormap(&tm_c);
    prefetch_tensormap(&tm_r);
  }
  __syncthreads();

  unsigned long long bar_target = 0;
  __shared__ int s_abort;  // SH: a cross-rank wait timed out (here or in another CTA of the rank)
  if (SH && tid == 0) s_abort = 0;
  // SH: the barrier's arrival, the flags and every system-scope fence are
  // done by warp 1 (thread 0 is the TMA producer: a fence there would wait
  // for its in-flight bulk copies)
  const int xt = tid - 32;
  auto gsync = [&](bool sysfence = false) {
    bar_target += (unsigned long long)G;
    if (!SH) {
      grid_barrier(&ctl->bar, bar_target);
      return;
    }
    __syncthreads();
    if (xt == 0) {
      // cumulative over every store this CTA's threads made before the
      // bar.sync above, including the ones into peer GPUs' inboxes: after
      // the barrier, CTA 0's system-scope flag release covers them all
      if (sysfence) asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&ctl->bar) : "memory");
      unsigned long long t0 = 0, v;
      // the abort checks (another CTA's fault flag, the timeout) run on every
      // 256th poll only: they add L2 traffic and latency to the spin
      for (unsigned spins = 0;; ++spins) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&ctl->bar) : "memory");
        if (v >= bar_target) break;
        if ((spins & 255u) == 255u) {
          if (t0 == 0) t0 = globaltimer_ns();
          if (*((volatile int32_t*)&ctl->fault) || globaltimer_ns() - t0 > kXchgTimeoutNs) {
            atomicExch(&ctl->fault, 2);
            s_abort = 1;
            break;
          }
        }
      }
    }
    __syncthreads();
  };

  // ---- the box sequence (identical walk on the producer and consumer side)
  auto plan_of = [&](int64_t k) -> const Plan& { return p.plan[k - p.k_begin]; };
  // this rank's rows of the iteration's row block (sharded: its interleaved
  // share, from the rank's range table; else the plan's global range)
  auto r_lo = [&](const Plan& pl) -> int { return SH ? (int)lrange[2 * pl.rb] : pl.r_lo; };
  auto r_hi = [&](const Plan& pl) -> int { return SH ? (int)lrange[2 * pl.rb + 1] : pl.r_hi; };
  auto cdiv = [](int a, int b) { return (a + b - 1) / b; };
  // TMA box columns start 16-byte aligned: a column block that starts on an
  // odd column is loaded from the even column before it (span = nJ + 1, the
  // extra leading column is weighted by zero / dropped)
  auto span_c = [](const Plan& pl) { return pl.c_hi - pl.c_lo + (pl.c_lo & 1); };
  // the row sweep runs `skew` steps behind the column sweep
  const int skew = p.extended ? 1 : 0;
  const int64_t s_end = p.k_end + skew;  // last step of this launch
  auto col_active = [&](int64_t s) { return p.extended && s <= p.k_end; };
  auto row_active = [&](int64_t s) { return s - skew >= p.k_begin; };
  // pass order within the two phases of a step (sp.order): 0 = C1 R1 | R2 C2
  // (R2 right behind R1: its 80 MB are still in L2), 1 = R1 C1 | C2 R2 (C2
  // right behind C1; R1's lines are loaded evict_last to survive the column
  // passes).  kind: 0 C1, 1 R1, 2 R2, 3 C2
  const int order = sp.order ? 1 : 0;
  auto kind_of = [&](int ph) -> int { return order ? (ph ^ 1) : ph; };
  // L2 policy per pass: R1 -> evict_last (R2 reads the same 80 MB right
  // after, across the two barriers), the column passes and R2 -> evict_first
  // (each byte is read once in the pass; keeping it would push R1's lines out
  // before R2)
  const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
  const int l2hint = sp.l2hint;
  // second passes (C2, R2) walk their row chunks last-to-first: the boxes the
  // first pass read most recently are the ones still in L2 (an LRU cache
  // re-read in the same order would miss on all of them)
  const bool rev = sp.reverse != 0;
  // C1's last `tail` row chunks are the first ones C2 (walking backwards)
  // reads again: they are loaded evict_last so they are still in L2 then
  const int tail = rev ? sp.tail : 0;

  // ---- producer (thread 0): the walk over the run's boxes as an incremental
  // state machine.  A pass is a nest of two counters (in: fastest); box
  // coordinates advance by per-pass steps, so issuing a box costs a handful
  // of instructions (no divisions, no plan lookups) on the consumers' critical
  // path; the per-pass setup runs four times per step.
  //   C1 (kind 0): subtile-major   (out = column subtile, in = row chunk; column sums run down the rows)
  //   C2 (kind 3): row-chunk-major (out = row chunk, in = subtile; row dots run across the subtiles)
  //   R1 (kind 1): row-chunk-major, R2 (kind 2): subtile-major
  struct Walk {
    int64_t k;   // step
    int ph;      // phase position 0..3 within the step
    int in, out, n_in, n_out;
    int x, y;              // coordinates of the next box
    int xb, yb;            // coordinates at (in, out) = (0, 0)
    int x_in, y_in, x_out, y_out;  // steps
    int keep_from;         // in >= keep_from: load evict_last (kind 0); INT_MAX: never; -1: always
    const CUtensorMap* map;
    uint32_t bytes;
  };
  Walk pw;
  pw.k = p.k_begin;
  pw.ph = -1;
  pw.n_in = pw.n_out = 0;
  pw.in = pw.out = 0;
  // set up the pass (k, ph); false if it has no boxes
  auto walk_setup = [&](Walk& w) -> bool {
    const int kd = kind_of(w.ph);
    w.in = w.out = 0;
    if (kd == 0 || kd == 3) {
      if (!col_active(w.k) || nR <= 0) return false;
      const Plan& pl = plan_of(w.k);
      const int nsc = cdiv(span_c(pl), cw), nrc = cdiv(nR, ch);
      const int x0 = (pl.c_lo & ~1), y0 = rbase + zr0;
      w.map = &tm_c;
      w.bytes = (uint32_t)(cw * ch * 8);
      if (kd == 0) {
        w.n_in = nrc, w.n_out = nsc;
        w.xb = x0, w.yb = y0;
        w.x_in = 0, w.y_in = ch, w.x_out = cw, w.y_out = 0;
        w.keep_from = tail > 0 ? nrc - tail : 0x7fffffff;
      } else {
        w.n_in = nsc, w.n_out = nrc;
        w.xb = x0, w.yb = rev ? y0 + (nrc - 1) * ch : y0;
        w.x_in = cw, w.y_in = 0, w.x_out = 0, w.y_out = rev ? -ch : ch;
        w.keep_from = 0x7fffffff;
      }
    } else {
      if (!row_active(w.k) || nC <= 0) return false;
      const Plan& pl = plan_of(w.k - skew);
      const int nsr = cdiv(nC, rw), nrr = cdiv(r_hi(pl) - r_lo(pl), rh);
      if (nrr <= 0) return false;
      const int x0 = xq0, y0 = rbase + r_lo(pl);
      w.map = &tm_r;
      w.bytes = (uint32_t)(rw * rh * 8);
      if (kd == 1) {
        w.n_in = nsr, w.n_out = nrr;
        w.xb = x0, w.yb = y0;
        w.x_in = rw, w.y_in = 0, w.x_out = 0, w.y_out = rh;
        w.keep_from = -1;
      } else {
        w.n_in = nrr, w.n_out = nsr;
        w.xb = x0, w.yb = rev ? y0 + (nrr - 1) * rh : y0;
        w.x_in = 0, w.y_in = rev ? -rh : rh, w.x_out = rw, w.y_out = 0;
        w.keep_from = 0x7fffffff;
      }
    }
    w.x = w.xb;
    w.y = w.yb;
    return w.n_in > 0 && w.n_out > 0;
  };
  // move to the next non-empty pass; k > s_end means the walk is over
  auto walk_next_pass = [&](Walk& w) {
    for (;;) {
      if (++w.ph == 4) {
        w.ph = 0;
        ++w.k;
      }
      if (w.k > s_end || walk_setup(w)) return;
    }
  };
  auto walk_advance = [&](Walk& w) {
    if (++w.in < w.n_in) {
      w.x += w.x_in;
      w.y += w.y_in;
      return;
    }
    w.in = 0;
    if (++w.out < w.n_out) {
      w.x = w.xb + w.out * w.x_out;
      w.y = w.yb + w.out * w.y_out;
      return;
    }
    walk_next_pass(w);
  };
  int pstage = 0;          // stage of the next issue
  int in_flight = 0;       // issued, not yet consumed
  auto refill = [&]() {    // thread 0: keep NS boxes in flight
    if (tid != 0) return;
    while (pw.k <= s_end && in_flight < NS) {
      // the stage was only READ by the generic proxy (ordered before this by
      // the take() barrier); a proxy fence is needed only for generic writes
      // the async proxy must see, so none here (REBK_STREAM_PFENCE=1 restores it)
      if (sp.pfence) fence_proxy_async();
      double* dst = sm + (size_t)pstage * SD;
      mbar_arrive_expect_tx(&sbar[pstage], pw.bytes);
      if (l2hint)
        tma_load_2d_hint(dst, pw.map, pw.x, pw.y, &sbar[pstage], pw.in >= pw.keep_from ? pol_last : pol_first);
      else
        tma_load_2d(dst, pw.map, pw.x, pw.y, &sbar[pstage]);
      if (++pstage == NS) pstage = 0;
      ++in_flight;
      walk_advance(pw);
    }
  };
  // consumer: wait for the next box, hand it to f, release its stage
  int cstage = 0;
  uint32_t cphase = 0;
  auto take = [&](auto f) {
    mbar_wait(&sbar[cstage], cphase);
    if (!(sp.dbg & 2)) f(sm + (size_t)cstage * SD);  // dbg 2: stream only (timing experiments)
    __syncthreads();  // every reader of this stage is done
    if (++cstage == NS) {
      cstage = 0;
      cphase ^= 1u;
    }
    --in_flight;
    refill();
  };

  const bool checking = p.stop_mode != 2;
  auto oracle_partial = [&]() {
    double acc = 0.0;
    for (int c = tid; c < nC; c += kStreamThreads) {
      const double d = s_x[c] - s_xs[c];
      acc = fma(d, d, acc);
    }
    const double s = block_sum<kStreamThreads>(acc, s_red);
    if (tid == 0) __stcg(errpart + g, s);
  };
  auto decide = [&](int64_t k) -> bool {
    if (warp == 0) {
      const double s = warp_sum_cg(errpart, G);
      if (lane == 0) s_bcast[0] = s;
    }
    __syncthreads();
    const double err = sqrt(s_bcast[0]);
    const bool conv = check_stops(err, p.tol, p.nonfinite_stop);
    if (g == 0 && tid == 0 && (!SH || vr == 0))
      record_check(ctl, p.errs, p.errs_cap, p.record, err, p.tol, p.nonfinite_stop, k);
    else if (SH && g == 0 && tid == 0 && check_stops(err, p.tol, p.nonfinite_stop)) {
      ctl->converged = err <= p.tol;  // the other virtual ranks: only what their CTAs read
      ctl->iters = k;
      ctl->done = 1;
    }
    __syncthreads();
    return conv;
  };

  // ---- cross-rank exchange (SH): publish, then wait for every rank's flag
  const unsigned long long seq_base = SH ? X.seq_base : 0ull;
  auto flag_at = [&](int q, int kind, int slot, int from, int cta) -> unsigned long long* {
    return X.flags[q] + (((int64_t)(kind * 2 + slot) * P + from) * G + cta);
  };
  // after this CTA's stores into the peers' inboxes: the bar.sync orders
  // every thread's stores before the flag stores, and a release at system
  // scope is cumulative over them (PTX memory model), so the peer that
  // acquires the flag sees the data
  auto publish = [&](int kind, int slot, int cta, unsigned long long seq) {
    __syncthreads();
    if (xt >= 0 && xt < P) st_release_sys_u64(flag_at(xt, kind, slot, rank, cta), seq);
  };
  auto await_all = [&](int kind, int slot, int cta, unsigned long long seq) {
    if (xt >= 0 && xt < P) {
      const unsigned long long* f = flag_at(rank, kind, slot, xt, cta);
      unsigned long long t0 = 0;
      for (unsigned spins = 0; ld_acquire_sys_u64(f) < seq; ++spins) {
        if ((spins & 255u) == 255u) {
          if (t0 == 0) t0 = globaltimer_ns();
          if (*((volatile int32_t*)&ctl->fault) || globaltimer_ns() - t0 > kXchgTimeoutNs) {
            atomicExch(&ctl->fault, 2);
            s_abort = 1;
            break;
          }
        }
      }
    }
    __syncthreads();
  };

  // Column sums of a box stream, subtile by subtile: out(c, Σ_r T[r][c] v[r])
  // for the C columns of subtile s; box rc holds rows [rc*bh, rc*bh + bh).
  // Threads own column pairs (cp) and a row residue (rg); the RG partials are
  // summed in fixed order through s_red.
  auto colsum_stream = [&](int C, int R, int bw, int bh, const double* v, bool rv, auto out) {
    const int nsub = cdiv(C, bw), nrc = cdiv(R, bh);
    for (int s = 0; s < nsub; ++s) {
      const int Cs = min(bw, C - s * bw);
      const int CP = (Cs + 1) >> 1;
      int RG = kStreamThreads / CP;
      if (RG > bh) RG = bh;
      const int cp = tid % CP, rg = tid / CP;
      double2 a0 = make_double2(0.0, 0.0), a1 = a0;
      for (int rci = 0; rci < nrc; ++rci) {
        const int rc = rv ? nrc - 1 - rci : rci;
        const int Rb = min(bh, R - rc * bh);
        const double* vb = v + rc * bh;
        take([&](const double* T) {
          if (rg < RG) {
            const double* col = T + 2 * cp;
            int r = rg;
            for (; r + RG < Rb; r += 2 * RG) {
              const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * bw);
              const double2 t1 = *reinterpret_cast<const double2*>(col + (size_t)(r + RG) * bw);
              const double v0 = vb[r], v1 = vb[r + RG];
              a0.x = fma(t0.x, v0, a0.x);
              a0.y = fma(t0.y, v0, a0.y);
              a1.x = fma(t1.x, v1, a1.x);
              a1.y = fma(t1.y, v1, a1.y);
            }
            if (r < Rb) {
              const double2 t0 = *reinterpret_cast<const double2*>(col + (size_t)r * bw);
              const double v0 = vb[r];
              a0.x = fma(t0.x, v0, a0.x);
              a0.y = fma(t0.y, v0, a0.y);
            }
          }
        });
      }
      if (rg < RG) {
        s_red[rg * 2 * CP + 2 * cp] = a0.x + a1.x;
        s_red[rg * 2 * CP + 2 * cp + 1] = a0.y + a1.y;
      }
      __syncthreads();
      for (int c = tid; c < Cs; c += kStreamThreads) {
        double acc = 0.0;
        for (int q = 0; q < RG; ++q) acc += s_red[q * 2 * CP + c];
        out(s * bw + c, acc);
      }
      __syncthreads();
    }
  };
  // Row dots of a box stream, row chunk by row chunk: out(r, Σ_c T[r][c] v[c])
  // over all subtiles of the row; L lanes per row (bh * L <= threads), the
  // accumulators carry across the subtiles of a row chunk.
  auto rowdot_stream = [&](int C, int R, int bw, int bh, int L, const double* v, bool rv, auto out) {
    const int nsub = cdiv(C, bw), nrc = cdiv(R, bh);
    const int sub = tid % L, rsub = tid / L;
    for (int rci = 0; rci < nrc; ++rci) {
      const int rc = rv ? nrc - 1 - rci : rci;
      const int Rb = min(bh, R - rc * bh);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      for (int s = 0; s < nsub; ++s) {
        const int Cs = min(bw, C - s * bw);
        const int CPf = Cs >> 1;
        const double* vs = v + s * bw;
        take([&](const double* T) {
          if (rsub < Rb) {
            const double2* row = reinterpret_cast<const double2*>(T + (size_t)rsub * bw);
            const double2* v2 = reinterpret_cast<const double2*>(vs);
            int q = sub;
            for (; q + L < CPf; q += 2 * L) {
              const double2 t0 = row[q], t1 = row[q + L];
              const double2 w0 = v2[q], w1 = v2[q + L];
              a0 = fma(t0.x, w0.x, a0);
              a1 = fma(t0.y, w0.y, a1);
              a2 = fma(t1.x, w1.x, a2);
              a3 = fma(t1.y, w1.y, a3);
            }
            if (q < CPf) {
              const double2 t0 = row[q], w0 = v2[q];
              a0 = fma(t0.x, w0.x, a0);
              a1 = fma(t0.y, w0.y, a1);
            }
            if ((Cs & 1) && sub == (CPf % L)) a2 = fma(T[(size_t)rsub * bw + Cs - 1], vs[Cs - 1], a2);
          }
        });
      }
      double acc = (a0 + a1) + (a2 + a3);
      for (int off = L / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (sub == 0 && rsub < Rb) out(rc * bh + rsub, acc);
      // out() writes are ordered before later readers by the next take()'s barrier
    }
  };

  long long prof_acc[16];
  for (int i = 0; i < 16; ++i) prof_acc[i] = 0;
  long long prof_last = clock64();
#define PROF(i)                          \
  if (p.prof) {                          \
    const long long _t = clock64();      \
    prof_acc[i] += _t - prof_last;       \
    prof_last = _t;                      \
  }
  bool finished = false;
  if (p.k_begin == 1 && checking) {
    oracle_partial();
    gsync();
    if (SH && s_abort) finished = true;
    else if (decide(0)) finished = true;
  }
  if (!finished) {
    if (tid == 0) walk_next_pass(pw);  // the first non-empty pass
    refill();
  }

  bool pending = false;
  int64_t pending_k = 0;
  bool stop_in_loop = false;  // stopped by a decision inside the loop: z is one column sweep ahead of x
  for (int64_t s = p.k_begin; !finished && s <= s_end; ++s) {
    const bool colact = col_active(s), rowact = row_active(s);
    const int64_t kr = s - skew;  // the row sweep's iteration
    const Plan plc = plan_of(colact ? s : kr);
    const Plan plr = plan_of(rowact ? kr : s);
    const int rl = r_lo(plr);
    const int nJ = plc.c_hi - plc.c_lo, nI = r_hi(plr) - rl;
    const int co = plc.c_lo & 1, W = nJ + co;  // column span of the boxes
    // exchange sequence numbers continue across solves (seq_base = the
    // exchanges of earlier solves), so a rank that starts the next solve
    // early writes the other slot than the one a slow peer may still read
    const unsigned long long seq_u = seq_base + (unsigned long long)s;
    const unsigned long long seq_x = seq_base + (unsigned long long)kr;
    const int slot_u = (int)(seq_u & 1), slot_x = (int)(seq_x & 1);
    const bool check_k = rowact && checking && (kr % p.stride == 0);
    PROF(0);
    // ---- X: C1(s) partial u over owned rows -> upart[e * G + g]
    auto pass_c1 = [&]() {
      if (!colact) return;
      if (nR > 0)
        colsum_stream(W, nR, cw, ch, s_z, false, [&](int c, double val) {
          if (c >= co) __stcg(upart + (int64_t)(c - co) * G + g, val);
        });
      else
        for (int c = tid; c < nJ; c += kStreamThreads) __stcg(upart + (int64_t)c * G + g, 0.0);
    };
    // R1(kr): partial r over owned columns -> rpart[e * G + g]
    auto pass_r1 = [&]() {
      if (!rowact) return;
      if (nC > 0)
        rowdot_stream(nC, nI, rw, rh, sp.lr, s_x, false,
                      [&](int r, double acc) { __stcg(rpart + (int64_t)r * G + g, acc); });
      else
        for (int r = tid; r < nI; r += kStreamThreads) __stcg(rpart + (int64_t)r * G + g, 0.0);
    };
    if (order == 0) {
      pass_c1();
      PROF(1);
      pass_r1();
    } else {
      pass_r1();
      PROF(1);
      pass_c1();
    }
    PROF(6);
    gsync();
    PROF(2);
    if (SH && s_abort) {
      finished = true;
      break;
    }
    if (pending) {
      pending = false;
      if (decide(pending_k)) {
        finished = true;
        stop_in_loop = true;
        break;
      }
    }
    if (colact) {
      for (int e = g * kStreamWarps + warp; e < nJ; e += G * kStreamWarps) {
        const double sum = warp_sum_cg(upart + (int64_t)e * G, G);
        if (lane == 0) {
          if (XCH) {
            for (int q = 0; q < P; ++q) __stcg(X.inbox_u[q] + ((int64_t)slot_u * P + rank) * X.nJ_cap + e, sum);
          } else {
            __stcg(gu + e, sum);
          }
        }
      }
    }
    PROF(3);
    if (rowact) {
      // r = (Σ partials - b_I) + z_kr[I]: gz holds z after column sweep kr
      // (C2 of this step starts only after the next barrier)
      for (int e = g * kStreamWarps + warp; e < nI; e += G * kStreamWarps) {
        const double sum = warp_sum_cg(rpart + (int64_t)e * G, G);
        if (lane == 0) {
          double rv = sum - __ldg(gb + rl + e);
          if (p.extended) rv += __ldcg(gz + rl + e);
          __stcg(gr + e, rv);
        }
      }
    }
    PROF(8);
    gsync(XCH && colact);  // exchanging: fence at system scope after the bar.sync (see gsync)
    if (SH && s_abort) {
      finished = true;
      break;
    }
    if (XCH && colact) {
      // the rank's u partial is complete in every inbox: CTA 0 raises the
      // flag, everyone waits for all P ranks', then sums in rank order
      if (g == 0 && xt >= 0 && xt < P) st_release_sys_u64(flag_at(xt, 0, slot_u, rank, 0), seq_u);
      await_all(0, slot_u, 0, seq_u);
      if (s_abort) {
        finished = true;
        break;
      }
    }
    PROF(4);
    // ---- Y: R2(kr)  x[xq] -= s_I · A[I, xq]ᵀ r
    const double rs = plr.r_scale;
    auto pass_r2 = [&]() {
      if (!rowact) return;
      for (int c = tid; c < nI; c += kStreamThreads) s_r[c] = __ldcg(gr + c);
      __syncthreads();
      if (!XCH) {
        if (nC > 0) colsum_stream(nC, nI, rw, rh, s_r, rev, [&](int c, double acc) { s_x[c] = s_x[c] - rs * acc; });
      } else {
        // this rank's column partials of A[I_p, xq]ᵀ r_p go to CTA g of every
        // rank (same column slice everywhere); the flags go up now, the sum
        // over ranks (finish_x) can wait until after C2: the exchange then
        // hides behind the z pass
        if (nC > 0) {
          if (nI > 0) {
            colsum_stream(nC, nI, rw, rh, s_r, rev, [&](int c, double acc) {
              for (int q = 0; q < P; ++q) __stcg(X.inbox_x[q] + ((int64_t)slot_x * P + rank) * X.n_cap + xq0 + c, acc);
            });
          } else {
            for (int c = tid; c < nC; c += kStreamThreads)
              for (int q = 0; q < P; ++q)
                __stcg(X.inbox_x[q] + ((int64_t)slot_x * P + rank) * X.n_cap + xq0 + c, 0.0);
          }
        }
        publish(1, slot_x, g, seq_x);
      }
      __syncthreads();
    };
    // C2(s): z[zr] -= s_J · A[zr, J] u
    auto pass_c2 = [&]() {
      if (!colact) return;
      for (int c = tid; c < W; c += kStreamThreads) {
        double uc = 0.0;
        if (c >= co) {
          if (XCH) {
            const double* ib = X.inbox_u[rank] + (int64_t)slot_u * P * X.nJ_cap + (c - co);
            for (int q = 0; q < P; ++q) uc += __ldcg(ib + (int64_t)q * X.nJ_cap);
          } else {
            uc = __ldcg(gu + c - co);
          }
        }
        s_u[c] = uc;
      }
      __syncthreads();
      const double cs = plc.c_scale;
      if (nR > 0)
        rowdot_stream(W, nR, cw, ch, sp.lc, s_u, rev, [&](int r, double acc) {
          const double zo = s_z[r];
          const double zn = zo - cs * acc;
          s_z[r] = zn;
          __stcg(gz + zr0 + r, zn);
          if (checking) __stcg(gzp + zr0 + r, zo);
        });
      // the last row chunk's s_z writes before the next step's C1 reads them
      // (within the pass, the next take()'s barrier orders them)
      __syncthreads();
    };
    if (order == 0) {
      pass_r2();
      PROF(10);
      pass_c2();
    } else {
      pass_c2();
      PROF(10);
      pass_r2();
    }
    PROF(5);
    if (rowact && XCH) {
      await_all(1, slot_x, g, seq_x);
      if (s_abort) {
        finished = true;
        break;
      }
      const double* ib = X.inbox_x[rank] + (int64_t)slot_x * P * X.n_cap + xq0;
      for (int c = tid; c < nC; c += kStreamThreads) {
        double acc = 0.0;
        for (int q = 0; q < P; ++q) acc += __ldcg(ib + (int64_t)q * X.n_cap + c);
        s_x[c] = s_x[c] - rs * acc;
      }
      __syncthreads();
    }
    PROF(12);
    if (sp.dbg & 1) gsync();
    if (check_k) {
      oracle_partial();
      pending = true;
      pending_k = kr;
    }
  }
  if (!finished) {
    if (pending) {
      gsync();
      if (decide(pending_k)) finished = true;
    }
    if (!finished && p.k_end == p.max_iters) {
      if (checking && (p.max_iters % p.stride) != 0) {
        oracle_partial();
        gsync();
        decide(p.max_iters);
      }
      if (g == 0 && tid == 0) {
        if (!ctl->converged) ctl->iters = p.max_iters;
        ctl->done = 1;
      }
    }
  }
  if (p.prof && tid == 0)
    for (int i = 0; i < 16; ++i) p.prof[(int64_t)blockIdx.x * 16 + i] = prof_acc[i];
#undef PROF
  for (int c = tid; c < nC; c += kStreamThreads) __stcg(gx + xq0 + c, s_x[c]);
  if (p.extended) {
    // a stop decided inside the loop is for x before the latest column sweep
    for (int r = tid; r < nR; r += kStreamThreads)
      __stcg(gz + zr0 + r, stop_in_loop ? __ldcg(gzp + zr0 + r) : s_z[r]);
  }
  // boxes issued for iterations past a stop are still landing: drain them
  // (in_flight is tracked by thread 0, the only issuer)
  if (tid == 0)
    while (in_flight > 0) {
      mbar_wait(&sbar[cstage], cphase);
      if (++cstage == NS) {
        cstage = 0;
        cphase ^= 1u;
      }
      --in_flight;
    }
  __syncthreads();
}

__global__ void __launch_bounds__(kStreamThreads, 1)
    rebk_dense_stream_kernel(const __grid_constant__ StreamParams sp, const __grid_constant__ CUtensorMap tm_c,
                             const __grid_constant__ CUtensorMap tm_r) {
  stream_body<false>(sp, tm_c, tm_r);
}

__global__ void __launch_bounds__(kStreamThreads, 1)
    rebk_shard_stream_kernel(const __grid_constant__ StreamParams sp, const __grid_constant__ CUtensorMap tm_c,
                             const __grid_constant__ CUtensorMap tm_r) {
  stream_body<true>(sp, tm_c, tm_r);
}

static cudaError_t set_stream_attrs() {
  static int configured_device = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured_device == dev) return cudaSuccess;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(rebk_dense_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(rebk_shard_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
  if (e == cudaSuccess) configured_device = dev;
  return e;
}

cudaError_t stream_kernel_occupancy(size_t smem_bytes, int* blocks_per_sm) {
  cudaError_t e = set_stream_attrs();
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, rebk_dense_stream_kernel, kStreamThreads,
                                                       smem_bytes);
}

cudaError_t launch_dense_stream(const StreamParams& sp, const CUtensorMap& tm_c, const CUtensorMap& tm_r, int G,
                                size_t smem_bytes, cudaStream_t stream) {
  cudaError_t e = set_stream_attrs();
  if (e != cudaSuccess) return e;
  StreamParams spc = sp;
  CUtensorMap a = tm_c, b = tm_r;
  void* args[] = {&spc, &a, &b};
  return cudaLaunchCooperativeKernel((const void*)rebk_dense_stream_kernel, dim3(G), dim3(kStreamThreads), args,
                                     smem_bytes, stream);
}

// Row-sharded launch: X.vranks * X.Gr CTAs (one rank per launch on a real
// multi-GPU job; every emulated rank's CTAs co-resident in one cooperative
// launch on a single GPU, so ranks that wait on each other always run together)
cudaError_t launch_shard_stream(const StreamParams& sp, const CUtensorMap& tm_c, const CUtensorMap& tm_r,
                                size_t smem_bytes, cudaStream_t stream) {
  cudaError_t e = set_stream_attrs();
  if (e != cudaSuccess) return e;
  StreamParams spc = sp;
  CUtensorMap a = tm_c, b = tm_r;
  void* args[] = {&spc, &a, &b};
  return cudaLaunchCooperativeKernel((const void*)rebk_shard_stream_kernel, dim3(sp.x.vranks * sp.x.Gr),
                                     dim3(kStreamThreads), args, smem_bytes, stream);
}

}  // namespace rebk

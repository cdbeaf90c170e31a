"""REABK benchmark (BASELINE.json metric), headline on BASELINE config 3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c1|c2|c4|c5]

A step is one full solve of the workload to ||x - x*|| <= 1e-6 ||x*|| (the
reference's run(), solvers.py:425-474).  The default workload is C3
(200000 x 10000 fp64, 16 GB: the largest BASELINE config that fits one
B200).  N = 1: the streaming kernel; `value` = iterations/s with A, b, x*
resident in HBM (rebk_run_device); `e2e` = the same metric through the
C-ABI from pinned host buffers (A re-uploaded every step).  N > 1
(torchrun): A row-sharded over the ranks, one strong-scaled solve per step
(SURVEY §8e), timed as the max over ranks.  The other workloads keep their
own arms (C1/C2/C4 replicas at N > 1).  `--impl reference` times the
reference's own CPU path (the installed, unmodified kaczmarz package in
baseline/_ref; the oracle port if absent) on the host cores on a bounded
sample of the same instance and prints the same `config` dict.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "REABK iterations/s"
UNIT = "iters/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def build_workload(name):
    from paper_2001_04179_b200 import workloads

    t0 = time.time()
    wl = workloads.build(name)
    log(f"[bench] built {name}: A {wl.problem.a.shape}, beta_max={wl.beta_max:.6g}, alpha={wl.alpha:.6g} "
        f"({time.time() - t0:.1f}s)")
    return wl


def workload_desc(name, wl):
    m, n = wl.problem.a.shape
    tr, tc = max(wl.row_partition.block_sizes()), max(wl.col_partition.block_sizes())
    desc = {
        "c1": "C1 dense fp64 2000x500 randn, inconsistent",
        "c2": "C2 dense fp64 4000x10000 rank 2000 (U diag(s) V^T, s~U[1,10]), inconsistent",
        "c4": "C4 sparse fp64 CSR 200000x50000, 1e7 nnz, inconsistent",
    }[name]
    a_bytes = (wl.problem.a.nnz * 12 * 2) if wl.problem.a.is_sparse else m * n * 8
    l2 = (f"inputs larger than L2: A = {a_bytes / 1e6:.0f} MB > 126 MB L2, no flush" if a_bytes > 126e6
          else f"A = {a_bytes / 1e6:.0f} MB is L2-resident (no flush; L2 roofline applies)")
    return {
        "workload": f"{desc}; row/col blocks {tr}/{tc}; alpha=1/beta_max; stop ||x-x*||/||x*||<1e-6; seed 17",
        "m": m, "n": n, "row_block": tr, "col_block": tc,
        "alpha": wl.alpha, "beta_max": wl.beta_max,
        "l2_policy": l2,
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception as exc:  # pragma: no cover
            log(f"[bench] nvidia-smi unavailable: {exc}")
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names[1:], parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": float(np.median(sm)) if sm else None,
            "sm_max_mhz": float(max(smax)) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measured_read_peaks():
    """L2 and HBM read bandwidth measured on this pool's B200 by
    tools/l2_bw.cu (profiles/r02_l2_bw.json): {buffer MB: GB/s}."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_l2_bw.json")) as fh:
            pts = json.load(fh)["points"]
        return {int(p["buffer_mb"]): float(p["read_gbs"]) for p in pts}
    except Exception:
        return {}


def l2_roofline(a_bytes):
    """(peak GB/s, source) of the L2 read bandwidth for an A of a_bytes, or
    None when A does not fit the 126 MB L2."""
    pts = measured_read_peaks()
    if a_bytes > 96e6 or not pts:
        return None
    mb = min((k for k in pts if k < 1000 and k * 2**20 >= a_bytes), default=None)
    if mb is None:
        return None
    return pts[mb], f"measured L2 read bandwidth, {mb} MB buffer (tools/l2_bw.cu, profiles/r02_l2_bw.json)"


def profiled_traffic(workload):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(workload)
    except Exception:
        return None


# ------------------------------------------------------------------ CPU arms
def reference_module():
    """The UNMODIFIED reference package, pip-installed into baseline/_ref
    (DESIGN.md §6); None when that install is absent (then the oracle port
    stands in, kind "port")."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(path, "kaczmarz", "solvers.py")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import kaczmarz

    return kaczmarz


def host_threads():
    """Use every host core for the reference's BLAS (OpenBLAS may cap it)."""
    ncpu = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=ncpu, user_api="blas")
    except Exception:
        pass
    return ncpu


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        n = [d.get("num_threads", 1) for d in threadpool_info() if d.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


class ReferenceSampler:
    """Times the reference's CPU path on a bounded sample of a workload.

    kind "reference": the installed reference (baseline/_ref) — one
    kaczmarz.prepare(problem, config) (setup, excluded like run()'s
    wall_time, solvers.py:446/:465), then per sample `iters` iterations of
    exactly run()'s loop body: ctx.step(state) and the oracle_error check
    ||x - x*|| (solvers.py:398-407, :449-458) every iteration, timed with
    perf_counter from the same start state.  kind "port": the oracle port
    (oracle/rebk_oracle.py, the reference's numpy operations) when the
    install is absent."""

    def __init__(self, a, b, x_star, row_ptr, col_ptr, alpha, beta, seed, tol, sparse=False):
        self.K = reference_module()
        self.ncpu = host_threads()
        self.tol, self.x_star = tol, np.asarray(x_star)
        t0 = time.perf_counter()
        if self.K is not None:
            K = self.K
            mat = K.Matrix.from_sparse(a) if sparse else K.Matrix.from_dense(a)
            prob = K.ProblemInstance(a=mat, b=np.asarray(b), x_star=self.x_star, b_perp=None,
                                     meta=K.ProblemMeta(0, None, False, 0, 0.0))
            blocks = lambda p: tuple(range(int(p[i]), int(p[i + 1])) for i in range(len(p) - 1))
            rp = K.Partition("row", int(row_ptr[-1]), blocks(row_ptr))
            cp = K.Partition("col", int(col_ptr[-1]), blocks(col_ptr))
            self.cfg = K.SolverConfig(algorithm="rebk", alpha=alpha, seed=seed, row_partition=rp, col_partition=cp,
                                      max_iters=50_000, stop=K.StoppingRule(tol=tol), beta_max=beta)
            self.ctx = K.prepare(prob, self.cfg)
            self.kind = "reference"
        else:
            from oracle.rebk_oracle import OracleSolver

            dense = a.toarray() if sparse else a
            self.orc = OracleSolver(dense, np.asarray(b), np.asarray(row_ptr), np.asarray(col_ptr), alpha, "rebk")
            self.seed = seed
            self.kind = "port"
        self.setup_s = time.perf_counter() - t0

    def sample(self, iters):
        """(iterations run, loop seconds) of the first `iters` iterations."""
        if self.kind == "port":
            from oracle.rebk_oracle import NumpyRng

            res = self.orc.run(self.seed, iters, self.tol, self.x_star, rng=NumpyRng(self.seed))
            return res["iters"], res["wall_time"]
        ctx, xs, tol = self.ctx, self.x_star, self.tol
        st = ctx.initial_state()
        t0 = time.perf_counter()
        k = 0
        if not np.linalg.norm(st.x - xs) <= tol:
            for k in range(1, iters + 1):
                ctx.step(st)
                if np.linalg.norm(st.x - xs) <= tol:
                    break
        return k, time.perf_counter() - t0

    def describe(self, iters, workload):
        what = ("the installed reference (baseline/_ref kaczmarz 0.1.0): prepare() once, then per sample the "
                "run() loop body (ctx.step + oracle_error check)" if self.kind == "reference" else
                "oracle port (the reference's numpy operations + numpy Philox)")
        return (f"first {iters} REBK iterations of the same {workload} instance per sample; {what}; "
                f"BLAS threads {blas_threads()} of {self.ncpu} host CPUs; setup (prepare) {self.setup_s:.1f} s "
                f"excluded")


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if args.workload == "c3":
        return run_reference_c3(args)
    if args.workload == "c5":
        return run_reference_c5(args)
    wl = build_workload(args.workload)
    sp = wl.problem.a.is_sparse
    samp = ReferenceSampler(wl.problem.a._csr if sp else wl.problem.a.to_dense(), wl.problem.b,
                            wl.problem.x_star, wl.row_partition.pointers(), wl.col_partition.pointers(), wl.alpha,
                            wl.beta_max, wl.seed, wl.rel_tol * float(np.linalg.norm(wl.problem.x_star)), sparse=sp)
    return reference_line(args, samp, args.ref_iters, workload_desc(args.workload, wl), ws)


def reference_line(args, samp, sample_iters, config, ws, metric=METRIC, unit=UNIT, per=1.0):
    for _ in range(args.warmup):
        samp.sample(min(sample_iters, 10))
    iters_tot, secs = 0, 0.0
    for _ in range(args.steps):
        it, s = samp.sample(sample_iters)
        iters_tot += it
        secs += s
    v = iters_tot / secs / per
    line = {
        "impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload == "c3" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config,
        "cpu_baseline": {"value": v, "unit": unit, "cores": blas_threads(), "host_cpus": os.cpu_count(),
                         "kind": samp.kind, "sample": samp.describe(sample_iters, args.workload)},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def c3_config(wl):
    """The config dict BOTH arms print for C3 (identical keys and values)."""
    m, n = wl.shape
    return {"workload": f"C3 dense fp64 {m}x{n} randn (16 GB), inconsistent (r in null(A^T), ||r|| = 0.1 ||A x*||); "
                        "row/col blocks 1000/500; alpha=1/beta_max; stop ||x-x*||/||x*||<1e-6; seed 17; "
                        "A row-sharded over the job's GPUs when N > 1",
            "m": m, "n": n, "row_block": 1000, "col_block": 500, "alpha": wl.alpha, "beta_max": wl.beta_max,
            "l2_policy": "inputs larger than L2: A = 16 GB, no flush"}


def run_reference_c3(args):
    """C3 on the host cores: the instance is built on the GPU exactly as the
    ours arm builds it (workloads.c3_device; harness only) and copied to host
    memory; the reference then runs on the CPU."""
    import torch

    from paper_2001_04179_b200.workloads import c3_device

    t0 = time.time()
    wl = c3_device(device=0)
    a_h = wl.a.cpu().numpy()
    b_h, xs_h = wl.b.cpu().numpy(), wl.x_star.cpu().numpy()
    config = c3_config(wl)
    tol = wl.rel_tol * float(np.linalg.norm(xs_h))
    row_ptr, col_ptr, alpha, beta, seed = wl.row_ptr, wl.col_ptr, wl.alpha, wl.beta_max, wl.seed
    del wl
    torch.cuda.empty_cache()
    log(f"[bench] c3 on host ({time.time() - t0:.1f}s)")
    samp = ReferenceSampler(a_h, b_h, xs_h, row_ptr, col_ptr, alpha, beta, seed, tol)
    log(f"[bench] reference prepare {samp.setup_s:.1f}s (kind {samp.kind})")
    return reference_line(args, samp, args.ref_iters_c3, config, dist_env()[0])


def run_reference_c5(args):
    from paper_2001_04179_b200 import compute_beta_max, contiguous_partition, Matrix
    from paper_2001_04179_b200.workloads import c5_arrays

    a32, b32, xs = c5_arrays()
    m, n = a32.shape
    a64 = a32.astype(np.float64)
    rp, cp = contiguous_partition(m, 256, "row"), contiguous_partition(n, 256, "col")
    beta = compute_beta_max(Matrix.from_dense(a64), rp, cp)[2]
    samp = ReferenceSampler(a64, b32[:, 0].astype(np.float64), xs[:, 0], rp.pointers(), cp.pointers(), 1.0 / beta,
                            beta, 17, 1e-4 * float(np.linalg.norm(xs[:, 0])))
    return reference_line(args, samp, 200, c5_config(beta), dist_env()[0],
                          metric=METRIC + " (64 RHS per iteration)", per=b32.shape[1])


def c5_config(beta):
    return {"workload": "C5 dense fp32 50000x5000, 64 RHS sharing one block sequence, blocks 256/256, "
                        "alpha=1/beta_max, stop per column ||x-x*||/||x*||<1e-4",
            "m": 50000, "n": 5000, "nrhs": 64, "row_block": 256, "col_block": 256, "beta_max": beta,
            "l2_policy": "inputs larger than L2: A = 1 GB (+1 GB transposed copy), no flush"}


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import ctypes

    import torch

    import paper_2001_04179_b200 as P
    from paper_2001_04179_b200 import _lib

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    wl = build_workload(args.workload)
    prob = wl.problem
    m, n = prob.a.shape
    cfg = wl.config(max_iters=args.max_iters)
    ctx = P.prepare(prob, cfg)
    key = _lib.philox_key(cfg.seed)
    tol = cfg.stop.tol
    c = ctx.make_cfg(stop_mode="oracle_error", tol=tol, stride=1, max_iters=cfg.max_iters, key=key)
    dm = prob.a.device(device=local)
    dev = torch.device("cuda", local)
    b_d = torch.from_numpy(prob.b).to(dev)
    xs_d = torch.from_numpy(np.asarray(prob.x_star)).to(dev)
    x_d = torch.zeros(n, dtype=torch.float64, device=dev)
    z_d = torch.empty(m, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    lib = _lib.load()

    def device_solve():
        with torch.cuda.stream(stream):
            x_d.zero_()
            z_d.copy_(b_d)
        tr = _lib.RebkTrace()
        rc = lib.rebk_run_device(dm.handle, ctypes.byref(c), ctypes.c_void_p(b_d.data_ptr()),
                                 ctypes.c_void_p(xs_d.data_ptr()), ctypes.c_void_p(x_d.data_ptr()),
                                 ctypes.c_void_p(z_d.data_ptr()), ctypes.c_void_p(stream.cuda_stream),
                                 ctypes.byref(tr))
        _lib.check(rc, "rebk_run_device")
        return tr

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        tr = device_solve()
    log(f"[bench] warm-up solve: ITER={tr.iters} converged={bool(tr.converged)} "
        f"loop={tr.loop_ms:.3f} ms grid={tr.grid_ctas} path={tr.kernel_path}")

    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    iters_total, loop_ms_total, launches = 0, 0.0, 0
    for _ in range(args.steps):
        tr = device_solve()
        iters_total += int(tr.iters)
        loop_ms_total += float(tr.loop_ms)
        launches += 2  # sample_plan_kernel + rebk_dense_kernel (single chunk: max_iters < 2^20)
    ev1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    iters_t = torch.tensor([float(iters_total)], dtype=torch.float64, device=dev)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(iters_t, op=dist.ReduceOp.SUM)
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = float(iters_t.item()) / (ms_max / 1e3)
    per_solve_iters = iters_total / args.steps

    # roofline of the dominant kernel (rebk_dense_kernel), from its own events
    bytes_per_iter = wl.algorithmic_bytes_per_iter
    kernel_ms = loop_ms_total / args.steps
    achieved = bytes_per_iter * per_solve_iters / (kernel_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    bound = "hbm"
    a_bytes = (prob.a.nnz * 12 * 2) if prob.a.is_sparse else m * n * 8
    l2 = l2_roofline(a_bytes)
    if l2 is not None:  # A stays in L2 between iterations (C1): the L2 roofline applies
        peak, peak_src = l2
        bound = "l2"
    tr_info = profiled_traffic(args.workload)
    traffic = None
    if isinstance(tr_info, dict) and tr_info.get("bytes_per_iter"):
        # per launch like `achieved`: the ncu per-iteration figure x the
        # iterations one launch of this run covers
        traffic = float(tr_info["bytes_per_iter"]) * per_solve_iters
    elif isinstance(tr_info, (int, float)):
        traffic = float(tr_info)

    # e2e through the public API from pinned host buffers, A re-uploaded each step
    e2e = None
    if not args.no_e2e:
        b_pin = torch.from_numpy(prob.b).pin_memory()
        xs_pin = torch.from_numpy(np.asarray(prob.x_star)).pin_memory()
        if prob.a.is_sparse:
            import scipy.sparse as sps

            csr = prob.a._csr
            pins = [torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for v in (csr.data, csr.indices,
                                                                                   csr.indptr)]
            mat = P.Matrix.from_sparse(sps.csr_matrix((pins[0].numpy(), pins[1].numpy(), pins[2].numpy()),
                                                      shape=csr.shape))
            a_bytes = int(csr.data.nbytes + csr.indices.nbytes + csr.indptr.nbytes)
        else:
            a_pin = torch.from_numpy(prob.a.to_dense()).pin_memory()
            mat = P.Matrix.from_dense(a_pin.numpy())
            assert mat.to_dense().ctypes.data == a_pin.data_ptr()
            a_bytes = int(m * n * 8)
        prob2 = P.ProblemInstance(a=mat, b=b_pin.numpy(), x_star=xs_pin.numpy(), b_perp=None, meta=prob.meta)
        cfg2 = wl.config(max_iters=args.max_iters)
        cfg2.row_partition, cfg2.col_partition = wl.row_partition, wl.col_partition
        P.run(prob2, cfg2)  # warm
        mat.release_device()
        barrier()
        t0 = time.perf_counter()
        e_iters = 0
        for _ in range(args.steps):
            tr2 = P.run(prob2, cfg2)
            e_iters += tr2.iters
            mat.release_device()
        barrier()
        e_s = time.perf_counter() - t0
        e_t = torch.tensor([e_s], dtype=torch.float64, device=dev)
        ei_t = torch.tensor([float(e_iters)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
            dist.all_reduce(ei_t, op=dist.ReduceOp.SUM)
        e2e = {
            "value": float(ei_t.item()) / float(e_t.item()), "unit": UNIT,
            "h2d_bytes_per_step": int(a_bytes + 2 * m * 8 + 2 * n * 8),
            "d2h_bytes_per_step": int((m + n) * 8 + 64),
            "time_to_tol_s": float(e_t.item()) / args.steps,
            "path": "paper_2001_04179_b200.run(problem, config): A, b, x* uploaded from pinned host memory "
                    "every step (fresh device ctx), x and z read back",
        }

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        sp = prob.a.is_sparse
        samp = ReferenceSampler(prob.a._csr if sp else prob.a.to_dense(), prob.b, prob.x_star,
                                wl.row_partition.pointers(), wl.col_partition.pointers(), wl.alpha, wl.beta_max,
                                wl.seed, tol, sparse=sp)
        it, s = samp.sample(args.ref_iters)
        cpu = {"value": it / s, "unit": UNIT, "cores": blas_threads(), "host_cpus": os.cpu_count(),
               "kind": samp.kind, "sample": samp.describe(it, args.workload) + f"; {s:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(args.workload, wl),
            "details": {"parallelism": f"replicas x{ws}", "iters_per_solve": per_solve_iters,
                        "grid_ctas": int(tr.grid_ctas),
                        "kernel_path": ["rebk_dense_kernel", "rebk_dense_fast_kernel (cluster)",
                                        "rebk_dense_fast_kernel (cluster, cooperative)",
                                        "rebk_csr_kernel", "", "",
                                        "rebk_dense_split_kernel (column/row groups)",
                                        "rebk_dense_stream_kernel (TMA ring)"][int(tr.kernel_path)]},
            "time_to_tol_s": ms_max / args.steps / 1e3,
            "achieved_gbps": achieved,
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_note": (tr_info or {}).get("note") if isinstance(tr_info, dict) else None,
                         "kernel": ["rebk_dense_kernel", "rebk_dense_fast_kernel", "rebk_dense_fast_kernel",
                                    "rebk_csr_kernel", "", "", "rebk_dense_split_kernel",
                                    "rebk_dense_stream_kernel"][int(tr.kernel_path)],
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_iter": bytes_per_iter,
                         "iters_per_launch": per_solve_iters, "kernel_ms_per_launch": kernel_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_ours_c5(args):
    """Config 5 (fp32, 64 RHS): value = REBK iterations/s of the whole batch
    (each iteration advances all 64 right-hand sides).  Kernel: the persistent
    tcgen05 whole-run kernel (rebk_mrhs_tc.cu)."""
    import torch

    from paper_2001_04179_b200 import contiguous_partition, SolverConfig, StoppingRule, Matrix, compute_beta_max
    from paper_2001_04179_b200.multirhs import DeviceMatrix32, run_multi
    from paper_2001_04179_b200.workloads import c5_arrays

    m, n, R, blk = 50000, 5000, 64, 256
    t0 = time.time()
    a32, b32, xs = c5_arrays()
    a64 = Matrix.from_dense(a32.astype(np.float64))
    rp, cp = contiguous_partition(m, blk, "row"), contiguous_partition(n, blk, "col")
    beta = compute_beta_max(a64, rp, cp)[2]
    log(f"[bench] built c5 ({time.time() - t0:.1f}s), beta_max={beta:.6g}")
    stride = int(os.environ.get("REBK_BENCH_STRIDE", "1"))
    cfg = SolverConfig(algorithm="rebk", alpha=1.0 / beta, seed=17, max_iters=args.max_iters, row_partition=rp,
                       col_partition=cp, stop=StoppingRule(tol=1.0, check_stride=stride), beta_max=beta)
    tols = 1e-4 * np.linalg.norm(xs, axis=0)
    dm = DeviceMatrix32(a32)
    tr = None
    for _ in range(max(args.warmup, 1)):
        tr = run_multi(a32, b32, cfg, X_star=xs, tols=tols, device_matrix=dm, a64=a64)
    log(f"[bench] c5 warm-up: K={tr.iters} per-RHS ITER {tr.iters_per_rhs.min()}..{tr.iters_per_rhs.max()} "
        f"loop {tr.wall_time * 1e3:.1f} ms path={tr.kernel_path}")
    clocks = ClockSampler(0)
    torch.cuda.synchronize()
    clocks.start()
    its, secs = 0, 0.0
    for _ in range(args.steps):
        tr = run_multi(a32, b32, cfg, X_star=xs, tols=tols, device_matrix=dm, a64=a64)
        its += tr.iters
        secs += tr.wall_time
    torch.cuda.synchronize()
    clk = clocks.stop()
    value = its / secs
    per_solve = its / args.steps
    # algorithmic bytes: the two selected fp32 blocks read once (nominal 256-wide blocks);
    # the iterates (Z, X read+write, 64 RHS) are reported separately
    bytes_per_iter = 4.0 * (m * blk + blk * n)
    vec_bytes_per_iter = 2 * 4.0 * R * (m + n)
    flops_per_iter = 2 * 2.0 * blk * R * m + 2 * 2.0 * blk * R * n
    achieved = bytes_per_iter * value / 1e9
    peak, peak_src = measured_peak()
    tr_info = profiled_traffic("c5")
    traffic = None
    if isinstance(tr_info, dict) and tr_info.get("bytes_per_iter"):
        traffic = float(tr_info["bytes_per_iter"]) * per_solve

    e2e = None
    if not args.no_e2e:
        a_pin = torch.from_numpy(a32).pin_memory()
        b_pin = torch.from_numpy(b32).pin_memory()
        xs_pin = torch.from_numpy(np.ascontiguousarray(xs, dtype=np.float32)).pin_memory()
        run_multi(a_pin.numpy(), b_pin.numpy(), cfg, X_star=xs_pin.numpy(), tols=tols)  # warm
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        e_its = 0
        for _ in range(args.steps):
            tr2 = run_multi(a_pin.numpy(), b_pin.numpy(), cfg, X_star=xs_pin.numpy(), tols=tols)
            e_its += tr2.iters
        torch.cuda.synchronize()
        e_s = time.perf_counter() - t1
        e2e = {"value": e_its / e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(4 * (m * n + m * R + n * R)),
               "d2h_bytes_per_step": int(4 * (n * R + m * R) + 16 * R),
               "time_to_tol_s": e_s / args.steps,
               "path": "paper_2001_04179_b200.multirhs.run_multi(A, B, config): A (1 GB fp32), B and X* uploaded "
                       "from pinned host memory every step (fresh fp32 device context incl. its transposed copy; "
                       "the sampler's block weights computed on the device from that copy, as the public API does "
                       "by default), X and Z read back"}

    cpu = None
    if not args.no_cpu:
        samp = ReferenceSampler(a64.to_dense(), b32[:, 0].astype(np.float64), xs[:, 0], rp.pointers(),
                                cp.pointers(), 1.0 / beta, beta, 17, 1e-300)
        it, s = samp.sample(200)
        cpu = {"value": it / s / R, "unit": UNIT, "cores": blas_threads(), "host_cpus": os.cpu_count(),
               "kind": samp.kind,
               "sample": samp.describe(it, "c5") + f" (right-hand side 0 in fp64: the reference solves one RHS "
                                                   f"per run, so 64 RHS per iteration = 64 such iterations); "
                                                   f"{s:.2f} s"}

    line = {
        "metric": METRIC + " (64 RHS per iteration)", "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (3xTF32 tcgen05)", "data": "synthetic",
        "config": c5_config(beta),
        "details": {"K": tr.iters, "check_stride": stride, "iters_per_solve": per_solve,
                    "kernel_path": "k_rebk_mrhs_persistent (tcgen05 kind::tf32, 3xTF32, TMEM accumulators)"},
        "time_to_tol_s": secs / args.steps,
        "achieved_gbps": achieved,
        "achieved_tflops": flops_per_iter * value / 1e12,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "k_rebk_mrhs_persistent", "peak_source": peak_src,
                     "algorithmic_bytes_per_iter": bytes_per_iter, "vector_bytes_per_iter": vec_bytes_per_iter,
                     "iters_per_launch": per_solve, "kernel_ms_per_launch": 1e3 * secs / args.steps,
                     "traffic_note": (tr_info or {}).get("note") if isinstance(tr_info, dict) else None},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": 10 * args.steps,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours_c3(args):
    """Config 3 (16 GB dense fp64) on one GPU, the N = 1 headline: instance
    built on the device, the streaming kernel through the device-pointer
    C-ABI (rebk_run_device).  e2e: A, b, x* uploaded from pinned host memory
    through rebk_ctx_create_dense + rebk_run (the C-ABI a reference-side
    binding calls) every step, x and z read back."""
    import ctypes

    import torch

    from paper_2001_04179_b200 import _lib
    from paper_2001_04179_b200.matrix import DeviceMatrix
    from paper_2001_04179_b200.workloads import c3_device

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    t0 = time.time()
    wl = c3_device(device=local)
    m, n = wl.shape
    log(f"[bench] built c3 on device: A {wl.shape}, beta_max={wl.beta_max:.6g} ({time.time() - t0:.1f}s)")
    dev = torch.device("cuda", local)
    lib = _lib.load()
    dm = DeviceMatrix.from_device_pointer(wl.a.data_ptr(), m, n, n, local)
    tol = wl.rel_tol * float(wl.x_star.norm())
    c = wl.cfg("oracle_error", tol, args.max_iters)
    x_d = torch.zeros(n, dtype=torch.float64, device=dev)
    z_d = torch.empty(m, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def device_solve():
        with torch.cuda.stream(stream):
            x_d.zero_()
            z_d.copy_(wl.b)
        tr = _lib.RebkTrace()
        _lib.check(lib.rebk_run_device(dm.handle, ctypes.byref(c), ctypes.c_void_p(wl.b.data_ptr()),
                                       ctypes.c_void_p(wl.x_star.data_ptr()), ctypes.c_void_p(x_d.data_ptr()),
                                       ctypes.c_void_p(z_d.data_ptr()), ctypes.c_void_p(stream.cuda_stream),
                                       ctypes.byref(tr)), "rebk_run_device")
        return tr

    for _ in range(max(args.warmup, 1)):
        tr = device_solve()
    log(f"[bench] c3 warm-up: ITER={tr.iters} converged={bool(tr.converged)} loop={tr.loop_ms:.1f} ms "
        f"path={tr.kernel_path}")
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    iters, loop_ms = 0, 0.0
    for _ in range(args.steps):
        tr = device_solve()
        iters += int(tr.iters)
        loop_ms += float(tr.loop_ms)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    value = iters / (ms / 1e3)
    per_solve = iters / args.steps
    kernel_ms = loop_ms / args.steps
    achieved = wl.algorithmic_bytes_per_iter * per_solve / (kernel_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    tr_info = profiled_traffic("c3")

    e2e = None
    cpu = None
    if not (args.no_e2e and args.no_cpu):
        a_pin = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
        a_pin.copy_(wl.a)
        b_h, xs_h = wl.b.cpu().numpy(), wl.x_star.cpu().numpy()
    if not args.no_e2e:
        x_h, z_h = np.empty(n), np.empty(m)
        b_pin = torch.from_numpy(b_h).pin_memory()
        xs_pin = torch.from_numpy(xs_h).pin_memory()
        x_pin = torch.empty(n, dtype=torch.float64).pin_memory()
        z_pin = torch.empty(m, dtype=torch.float64).pin_memory()

        def e2e_step():
            h = ctypes.c_void_p()
            _lib.check(lib.rebk_ctx_create_dense(ctypes.cast(ctypes.c_void_p(a_pin.data_ptr()),
                                                             ctypes.POINTER(ctypes.c_double)), m, n, n, local,
                                                 ctypes.byref(h)), "rebk_ctx_create_dense")
            tr2 = _lib.RebkTrace()
            p = lambda t: ctypes.cast(ctypes.c_void_p(t.data_ptr()), ctypes.POINTER(ctypes.c_double))
            _lib.check(lib.rebk_run(h, ctypes.byref(c), p(b_pin), None, None, p(xs_pin), p(x_pin), p(z_pin),
                                    ctypes.byref(tr2)), "rebk_run")
            lib.rebk_ctx_destroy(h)
            return int(tr2.iters)

        e2e_step()  # warm
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        e_iters = 0
        for _ in range(args.steps):
            e_iters += e2e_step()
        e_s = time.perf_counter() - t1
        e2e = {"value": e_iters / e_s, "unit": UNIT, "h2d_bytes_per_step": int(m * n * 8 + (m + n) * 8),
               "d2h_bytes_per_step": int((m + n) * 8), "time_to_tol_s": e_s / args.steps,
               "path": "rebk_ctx_create_dense (A from pinned host memory, 16 GB H2D) + rebk_run (host b, x*; x, z "
                       "read back) + rebk_ctx_destroy per step; the sampler arrays (block weights, cumulative "
                       "sums, alpha/w) are inputs of the C-ABI, computed once like the reference's SolverContext"}
        del x_h, z_h
    if not args.no_cpu:
        samp = ReferenceSampler(a_pin.numpy(), b_h, xs_h, wl.row_ptr, wl.col_ptr, wl.alpha, wl.beta_max, wl.seed, tol)
        it, s = samp.sample(args.ref_iters_c3)
        cpu = {"value": it / s, "unit": UNIT, "cores": blas_threads(), "host_cpus": os.cpu_count(),
               "kind": samp.kind, "sample": samp.describe(it, "c3") + f"; {s:.1f} s"}
        del samp

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (torch Philox on device)",
        "config": c3_config(wl),
        "details": {"parallelism": "1 GPU", "iters_per_solve": per_solve, "grid_ctas": int(tr.grid_ctas),
                    "kernel_path": "rebk_dense_stream_kernel (TMA ring)" if tr.kernel_path == 7 else str(tr.kernel_path)},
        "time_to_tol_s": ms / args.steps / 1e3,
        "achieved_gbps": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (float(tr_info["bytes_per_iter"]) * per_solve if isinstance(tr_info, dict) else None),
                     "traffic_note": (tr_info or {}).get("note"),
                     "kernel": "rebk_dense_stream_kernel",
                     "peak_source": peak_src, "algorithmic_bytes_per_iter": wl.algorithmic_bytes_per_iter,
                     "iters_per_launch": per_solve, "kernel_ms_per_launch": kernel_ms,
                     "two_pass_cap": two_pass_cap(wl),
                     "note": "the 800 MB column block cannot stay on chip between the u sum and the z update, so it "
                             "is read twice per iteration: frac <= two_pass_cap by construction",
                     "read_peak_gbs": measured_read_peaks().get(4096),
                     "read_peak_note": "pure-read HBM bandwidth measured by tools/l2_bw.cu (4 GB buffer); this kernel "
                                       "only reads A, so this is the tighter ceiling for it"},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": 2 * args.steps, "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    return 0


def two_pass_cap(wl):
    """Largest reachable frac for C3 on one GPU: algorithmic (read-once)
    bytes over the bytes that must move (column block twice, row block once)."""
    m, n = wl.shape
    tj = int(np.diff(wl.col_ptr).max())
    ti = int(np.diff(wl.row_ptr).max())
    return (m * tj + ti * n) / (2.0 * m * tj + ti * n)


def run_ours_c3_sharded(args):
    """Config 3 row-sharded over the job's GPUs: one
    process per GPU; every rank builds the same device instance and keeps its
    interleaved rows of every row block.  One persistent kernel per rank per
    solve (rebk_shard_stream_kernel): the |J|-length column products and the
    n-length x-update partials are exchanged INSIDE the kernel through peer
    memory (CUDA IPC over NVLink) with system-scope release flags, summed in
    rank order on every rank.  Strong scaling: the whole job does one solve
    per step.  `--python-loop` / `--nccl-driver` select the earlier
    host-driven variants (per-rank kernels + ncclAllReduce per iteration)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2001_04179_b200 import _lib
    from paper_2001_04179_b200.matrix import DeviceMatrix
    from paper_2001_04179_b200.sharded import (CudaShardBackend, NcclComm, ShardExchange, ShardPlan, nccl_unique_id,
                                                owned_rows, run_sharded_chunked, run_sharded_native)
    from paper_2001_04179_b200.workloads import c3_device

    ws, rank, local = dist_env()
    # NCCL prints its version banner on the C-level stdout; keep stdout for
    # the one JSON line by pointing fd 1 at stderr until the line is written
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if ws == 1 and "MASTER_ADDR" not in os.environ:
            import socket

            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(sk.getsockname()[1])
            sk.close()
        dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t0 = time.time()
    wl = c3_device(device=local)
    m, n = wl.shape
    abytes = wl.algorithmic_bytes_per_iter
    config = c3_config(wl)
    rows, ranges = owned_rows(wl.row_ptr, ws, rank)
    rows_t = torch.from_numpy(rows).to(dev)
    a_local = wl.a.index_select(0, rows_t).contiguous()
    b_local = wl.b.index_select(0, rows_t).contiguous()
    wl.a = None
    torch.cuda.empty_cache()
    tol = wl.rel_tol * float(wl.x_star.norm())
    log(f"[bench] c3 sharded rank {rank}/{ws}: {rows.size} rows of {m} ({time.time() - t0:.1f}s)")
    host_driver = args.python_loop or args.nccl_driver
    stream = torch.cuda.Stream(device=dev)
    x_d = torch.zeros(n, dtype=torch.float64, device=dev)
    z_d = torch.empty_like(b_local)
    fallback_reason = None
    xchg = dm = comm = None
    if not host_driver:
        # the in-kernel exchange; if its setup or first solve fails on any
        # rank (e.g. CUDA IPC refused), every rank falls back to the
        # host-driven NCCL loop and the line says so
        ok = 1
        try:
            c = wl.cfg("oracle_error", tol, args.max_iters)
            xchg = ShardExchange(ws, rank, int(np.diff(wl.col_ptr).max()), n, local, dist.all_gather_object)
            xchg.probe(dist.barrier)  # peer stores arrive before any kernel waits on them
            dm = DeviceMatrix.from_device_pointer(a_local.data_ptr(), a_local.shape[0], n, n, local)
            with torch.cuda.stream(stream):
                x_d.zero_()
                z_d.copy_(b_local)
            xchg.run(dm, c, ranges, b_local.data_ptr(), wl.x_star.data_ptr(), x_d.data_ptr(), z_d.data_ptr(),
                     stream.cuda_stream)
        except Exception as exc:  # pragma: no cover - exercised only on a failing multi-GPU box
            ok = 0
            fallback_reason = f"rank {rank}: {type(exc).__name__}: {exc}"
            log(f"[bench] in-kernel exchange unavailable, falling back to the NCCL driver: {fallback_reason}")
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            host_driver = True
            fallback_reason = fallback_reason or "another rank's in-kernel exchange failed"
    if host_driver:
        c = wl.cfg("max_iters_only", 1.0, args.max_iters)
        picks = np.empty((args.max_iters, 2), dtype=np.int32)
        _lib.check(_lib.load().rebk_sample_sequence(ctypes.byref(c), 1, args.max_iters,
                                                    picks.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))),
                   "rebk_sample_sequence")
        plan = ShardPlan(wl.row_ptr, wl.col_ptr, wl.alpha / wl.row_w, wl.alpha / wl.col_w, picks)
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = NcclComm(uid[0], ws, rank, local)

    def solve():
        if host_driver:
            be = CudaShardBackend.from_device(a_local, b_local, wl.x_star, True, local)
            if args.python_loop:
                res = run_sharded_chunked(be, plan, ranges, args.max_iters, tol,
                                          allreduce=lambda v: dist.all_reduce(v), chunk=32)
            else:
                res = run_sharded_native(be, comm, plan, ranges, args.max_iters, tol, chunk=32)
            return int(res["iters"]), bool(res["converged"]), float("nan")
        with torch.cuda.stream(stream):
            x_d.zero_()
            z_d.copy_(b_local)
        tr = xchg.run(dm, c, ranges, b_local.data_ptr(), wl.x_star.data_ptr(), x_d.data_ptr(), z_d.data_ptr(),
                      stream.cuda_stream)
        return int(tr.iters), bool(tr.converged), float(tr.loop_ms)

    for _ in range(max(args.warmup, 1)):
        it, conv, _ = solve()
    log(f"[bench] c3 sharded warm-up: ITER={it} converged={conv}")
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    iters, loop_ms = 0, 0.0
    for _ in range(args.steps):
        it, conv, lm = solve()
        iters += it
        loop_ms += lm
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    el = torch.tensor([ev0.elapsed_time(ev1) / 1e3, loop_ms / 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    secs, kernel_s = float(el[0].item()), float(el[1].item())
    value = iters / secs
    per_solve = iters / args.steps
    peak, peak_src = measured_peak()
    achieved = abytes * per_solve / (kernel_s / args.steps) / 1e9 if kernel_s > 0 else abytes * value / 1e9

    e2e = None
    if not args.no_e2e and not host_driver:
        # e2e per rank through the C-ABI: this rank's rows of A, b, x* from
        # pinned host memory into a fresh ctx, one sharded solve, x and z back
        a_pin = torch.empty(tuple(a_local.shape), dtype=torch.float64, pin_memory=True)
        a_pin.copy_(a_local)
        b_pin = b_local.cpu().pin_memory()
        xs_pin = wl.x_star.cpu().pin_memory()
        x_pin = torch.empty(n, dtype=torch.float64).pin_memory()
        z_pin = torch.empty(b_local.shape[0], dtype=torch.float64).pin_memory()
        lib = _lib.load()

        def e2e_step():
            h = ctypes.c_void_p()
            _lib.check(lib.rebk_ctx_create_dense(ctypes.cast(ctypes.c_void_p(a_pin.data_ptr()),
                                                             ctypes.POINTER(ctypes.c_double)), a_pin.shape[0], n, n,
                                                 local, ctypes.byref(h)), "rebk_ctx_create_dense")
            with torch.cuda.stream(stream):
                b2 = b_pin.to(dev, non_blocking=True)
                xs2 = xs_pin.to(dev, non_blocking=True)
                x2 = torch.zeros(n, dtype=torch.float64, device=dev)
                z2 = b2.clone()
            tr2 = _lib.RebkTrace()
            _lib.check(lib.rebk_shard_run_device(h, xchg.handle, ctypes.byref(c), _lib.i64ptr(np.ascontiguousarray(
                ranges, dtype=np.int64)), ctypes.c_void_p(b2.data_ptr()), ctypes.c_void_p(xs2.data_ptr()),
                ctypes.c_void_p(x2.data_ptr()), ctypes.c_void_p(z2.data_ptr()), ctypes.c_void_p(stream.cuda_stream),
                ctypes.byref(tr2)), "rebk_shard_run_device")
            with torch.cuda.stream(stream):
                x_pin.copy_(x2, non_blocking=True)
                z_pin.copy_(z2, non_blocking=True)
            stream.synchronize()
            lib.rebk_ctx_destroy(h)
            return int(tr2.iters)

        e2e_step()
        dist.barrier()
        t1 = time.perf_counter()
        e_iters = 0
        for _ in range(args.steps):
            e_iters += e2e_step()
        e_t = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device=dev)
        dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
        e_s = float(e_t.item())
        e2e = {"value": e_iters / e_s, "unit": UNIT,
               "h2d_bytes_per_step": int((m * n + m + ws * n) * 8), "d2h_bytes_per_step": int((m + ws * n) * 8),
               "time_to_tol_s": e_s / args.steps,
               "path": "per rank: rebk_ctx_create_dense (its rows of A from pinned host memory) + b, x* H2D + "
                       "rebk_shard_run_device + x, z D2H; job time = max over ranks (host clock around the "
                       "synchronous steps)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (torch Philox on device)",
            "config": config,
            "details": {"parallelism": f"row-sharded x{ws} (interleaved rows of every row block)",
                        "iters_per_solve": per_solve,
                        "timing": "CUDA events around the steps on each rank's stream, max over ranks",
                        "driver": ("python loop + torch.distributed NCCL" if args.python_loop else
                                   "rebk_shard_run (C++ issue loop, ncclAllReduce per iteration)" if host_driver else
                                   "rebk_shard_stream_kernel: one persistent kernel per rank per solve, u and dx "
                                   "exchanged in-kernel through peer memory (CUDA IPC) with release flags"),
                        "grid_ctas_per_rank": int(getattr(xchg, "grid_ctas", 0)) if not host_driver else None,
                        "fallback_reason": fallback_reason},
            "time_to_tol_s": secs / args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * ws, "unit": "GB/s",
                         "frac": achieved / (peak * ws), "traffic": None,
                         "kernel": "rebk_shard_stream_kernel (per rank)" if not host_driver else "rebk_shard_*",
                         "peak_source": peak_src + f" x {ws} GPUs",
                         "algorithmic_bytes_per_iter": abytes, "iters_per_launch": per_solve,
                         "kernel_ms_per_launch": 1e3 * kernel_s / args.steps},
            "cpu_baseline": None, "e2e": e2e,
            "gpu_launches": (8 * iters) if host_driver else 2 * args.steps, "clocks": clk,
        }
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    dist.barrier()
    for obj in (comm, dm, xchg):
        if obj is not None:
            obj.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="BASELINE config; c3 (the largest config that fits one B200) is the headline")
    ap.add_argument("--max-iters", type=int, default=50_000)
    ap.add_argument("--ref-iters", type=int, default=2000, help="iterations per CPU reference sample (c1/c2/c4)")
    ap.add_argument("--ref-iters-c3", type=int, default=100,
                    help="iterations per CPU reference sample (c3): ~2 s of host work each at ~50 iters/s")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="c3: row-sharded path also at N = 1")
    ap.add_argument("--python-loop", action="store_true", help="--sharded: issue each iteration from Python")
    ap.add_argument("--nccl-driver", action="store_true",
                    help="--sharded: the C++ issue loop with ncclAllReduce per iteration instead of the in-kernel exchange")
    args = ap.parse_args()
    ws = dist_env()[0]
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload == "c5":
        return run_ours_c5(args)
    if args.workload == "c3":
        # N > 1 (torchrun): A row-sharded over the ranks (strong scaling)
        return run_ours_c3_sharded(args) if (args.sharded or ws > 1) else run_ours_c3(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

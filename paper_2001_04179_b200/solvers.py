"""REBK and its row/column-sweep relatives on the B200, behind the reference's
solver interface.

Drop-in for ``kaczmarz.solvers`` (solvers.py): same ``run(problem, config)
-> RunTrace``, ``prepare(problem, config) -> SolverContext``,
``ctx.initial_state()`` / ``ctx.step(state)``, the same dataclasses and the
same validation errors.  The iteration itself never runs in Python:

* ``run`` hands the whole loop (solvers.py:425-474) to ``rebk_run`` in
  librebk.so: one persistent sm_100a kernel samples the block indices from
  the reference's Philox stream, applies the column and row sweeps and
  evaluates the stopping rule on the device.
* ``step`` (the per-iteration entry the reference's tests drive,
  solvers.py:267-268) draws the two uniforms from ``state.rng`` on the host
  exactly like the reference (so ScriptedRng works), then runs one device
  iteration with those explicit picks.

Algorithms on the device: rebk, rek, rabk, rk (step_rebk/step_rek/
step_rabk/step_rk, solvers.py:306-342) and dsbgs (step_dsbgs,
solvers.py:371-381: the joint submatrix sampler, with the reference's own
tables as inputs).  rbk and rdbk validate like the reference but raise
NotImplementedError: they apply per-block pseudoinverses (a different
kernel, outside this hot path).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import os

import numpy as np

from . import _lib
from .matrix import Matrix
from .problems import ProblemInstance
from .sampling import Partition, Rng, build_sampler, contiguous_partition, singleton_partition

ALGORITHMS = ("rk", "rek", "rbk", "rdbk", "rabk", "dsbgs", "rebk")

_EXTENDED = frozenset({"rek", "rdbk", "rebk"})
_NEEDS_COL_PARTITION = frozenset({"rdbk", "dsbgs", "rebk"})
_PROJECTION = frozenset({"rbk", "rdbk"})
_STEPSIZE_RATE_ALGOS = frozenset({"rk", "rek", "rabk", "rebk"})
DEVICE_ALGORITHMS = frozenset({"rk", "rek", "rabk", "rebk", "dsbgs"})

OutOfRegimeWarning = "stepsize at or beyond 2/beta_max: outside the guaranteed mean-square regime"


@dataclass
class StoppingRule:
    """When a run counts as converged (solvers.py:50-70)."""

    mode: str = "oracle_error"
    tol: float = 1e-5
    check_stride: int = 1

    def __post_init__(self):
        if self.mode not in ("oracle_error", "residual_proxy", "max_iters_only"):
            raise ValueError(f"unknown stopping mode {self.mode!r}")
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")
        if self.check_stride < 1:
            raise ValueError("check_stride must be at least 1")


@dataclass
class SolverConfig:
    algorithm: str
    alpha: float = 1.0
    row_partition: Partition | None = None
    col_partition: Partition | None = None
    seed: int = 0
    max_iters: int = 1_000_000
    stop: StoppingRule = field(default_factory=StoppingRule)
    x0: np.ndarray | None = None
    z0: np.ndarray | None = None
    record_errors: bool = False
    beta_max: float | None = None


@dataclass
class SolverState:
    x: np.ndarray
    z: np.ndarray | None
    k: int
    rng: Rng


@dataclass
class RunTrace:
    """Outcome of one run (solvers.py:96-112).  ``wall_time`` is the device
    time of the iteration loop (CUDA events), setup excluded as in the
    reference.  ``x``/``z`` carry the final iterates (the reference keeps them
    inside run(); exposing them costs nothing here)."""

    iters: int
    converged: bool
    wall_time: float
    final_error: float | None
    errors: np.ndarray | None = None
    checkpoints: np.ndarray | None = None
    warnings: tuple[str, ...] = ()
    x: np.ndarray | None = None
    z: np.ndarray | None = None
    grid_ctas: int = 0
    kernel_path: int = 0  # rebk_trace.kernel_path (include/rebk.h)
    # first check whose error was NaN/Inf (None: none).  The reference has no
    # finiteness check in run() and keeps iterating to max_iters; so does
    # this path (rebk_cfg.nonfinite_stop = 0), it only reports where
    nonfinite_at: int | None = None


def _block_beta(a: Matrix, p: Partition) -> float:
    """max over blocks of sigma_1(block)^2 / ||block||_F^2 (rates.py:76-90),
    via the eigenvalues of the smaller block Gram matrix."""
    worst = 0.0
    for idx in p.blocks:
        if len(idx) == 1:
            worst = max(worst, 1.0)
            continue
        view = a.block(p.axis, idx)
        fro = a.block_frobenius_sq(view)
        if fro <= 0.0:
            raise ValueError("zero block has no spectral-to-Frobenius ratio")
        blk = view.materialize()
        blk = blk.toarray() if hasattr(blk, "toarray") else np.asarray(blk)
        gram = blk @ blk.T if blk.shape[0] <= blk.shape[1] else blk.T @ blk
        worst = max(worst, float(np.linalg.eigvalsh(gram)[-1]) / fro)
    return worst


def compute_beta_max(a: Matrix, row_p: Partition, col_p: Partition) -> tuple[float, float, float]:
    br, bc = _block_beta(a, row_p), _block_beta(a, col_p)
    return br, bc, max(br, bc)


def _device_block_beta(a: Matrix, p: Partition, weights=None) -> float:
    """Same quantity as _block_beta (rates.py:76-90) with the spectral norms
    from device Lanczos on the immutable device copy of A (rebk_beta.cu).
    The Frobenius denominators are the host block norms the samplers use
    (matrix.py:170-189), so the ratio differs from the host one only by the
    eigenvalue solver's rounding."""
    sizes = np.array([len(idx) for idx in p.blocks])
    fro = np.asarray(weights if weights is not None else
                     [a.block_frobenius_sq(a.block(p.axis, idx)) for idx in p.blocks], dtype=np.float64)
    if np.any(fro <= 0.0):
        raise ValueError("zero block has no spectral-to-Frobenius ratio")
    worst = 1.0 if np.any(sizes == 1) else 0.0
    if np.all(sizes == 1):
        return worst
    order = None if p.is_contiguous_in_order() else p.order()
    dm = a.device(order, None) if p.axis == "row" else a.device(None, order)
    sig, _ = dm.block_sigma1_sq(0 if p.axis == "row" else 1, p.pointers())
    multi = sizes > 1
    return max(worst, float(np.max(sig[multi] / fro[multi])))


def device_beta_max(a: Matrix, row_p: Partition, col_p: Partition, row_w=None, col_w=None) -> tuple[float, float, float]:
    """compute_beta_max with the block spectral norms computed on the B200
    (dense A).  Sparse matrices keep the host eigensolver."""
    if a.is_sparse:
        return compute_beta_max(a, row_p, col_p)
    br, bc = _device_block_beta(a, row_p, row_w), _device_block_beta(a, col_p, col_w)
    return br, bc, max(br, bc)


class SolverContext:
    """Validated, immutable per-run data (solvers.py:123-187) plus the device
    binding: the device copy of A (permuted once when a partition is not
    contiguous) and the sampler arrays librebk consumes."""

    def __init__(self, problem: ProblemInstance, config: SolverConfig):
        algo = config.algorithm.lower()
        if algo not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {config.algorithm!r}")
        if config.alpha <= 0.0:
            raise ValueError("alpha must be positive")
        if algo in _PROJECTION and config.alpha != 1.0:
            raise ValueError(f"{algo} applies exact projections and has no stepsize")
        if config.max_iters < 0:
            raise ValueError("max_iters must be nonnegative")

        self.problem = problem
        self.config = config
        self.algorithm = algo
        self.a = problem.a
        self.b = np.asarray(problem.b, dtype=np.float64)
        if self.b.shape != (self.a.rows,):
            raise ValueError("right-hand side length does not match the matrix")
        self.alpha = float(config.alpha)
        self.extended = algo in _EXTENDED

        row_p = self._resolve_partition(config.row_partition, "row", self.a.rows)
        self.row_partition = row_p
        # start the H2D copy of A only once the run is known to go to the
        # device and the column partition has validated (a run that will
        # raise must not leave a copy of A behind); the validation is
        # repeated below in the reference's order, so error texts and
        # their precedence are unchanged
        needs_col = algo in _NEEDS_COL_PARTITION or algo == "rek"
        if algo in DEVICE_ALGORITHMS:
            try:
                early_col = self._resolve_partition(config.col_partition, "col", self.a.cols) if needs_col else None
            except ValueError:
                pass
            else:
                self._prefetch_device(row_p, early_col)
        self.row_sampler = build_sampler(self.a, row_p)
        self.row_scales = [float(self.alpha / w) for w in self.row_sampler.weights]
        self.row_selectors = [slice(i.start, i.stop) if isinstance(i, range) else i for i in row_p.blocks]

        self.col_partition = None
        self.col_sampler = None
        self.col_scales = None
        self.col_selectors = None
        if algo in _NEEDS_COL_PARTITION or algo == "rek":
            col_p = self._resolve_partition(config.col_partition, "col", self.a.cols)
            self.col_partition = col_p
            self.col_sampler = build_sampler(self.a, col_p)
            self.col_scales = [float(self.alpha / w) for w in self.col_sampler.weights]
            self.col_selectors = [slice(i.start, i.stop) if isinstance(i, range) else i for i in col_p.blocks]

        self.dsbgs_conditionals = None
        self.dsbgs_scales = None
        if algo == "dsbgs":
            self._build_dsbgs_tables()

        if algo not in DEVICE_ALGORITHMS:
            raise NotImplementedError(f"{algo} is not on the B200 hot path (it needs per-block pseudoinverses)")

        self.warnings: list[str] = []
        self.beta_max = config.beta_max
        if self.beta_max is None and algo in _STEPSIZE_RATE_ALGOS:
            col_p = self.col_partition or singleton_partition(self.a.cols, "col")
            col_w = self.col_sampler.weights if self.col_partition is not None else None
            # device Lanczos by default; REBK_BETA_BACKEND=host selects the host
            # eigensolver explicitly (prepare-only use on a machine without a GPU)
            backend = os.environ.get("REBK_BETA_BACKEND", "device")
            if backend not in ("device", "host"):
                raise ValueError(f"REBK_BETA_BACKEND must be 'device' or 'host', got {backend!r}")
            if backend == "device":
                self.beta_max = device_beta_max(self.a, row_p, col_p, self.row_sampler.weights, col_w)[2]
            else:
                self.beta_max = compute_beta_max(self.a, row_p, col_p)[2]
        if self.beta_max is not None and self.alpha >= 2.0 / self.beta_max:
            self.warnings.append(OutOfRegimeWarning)

        self._bind_device()

    def _build_dsbgs_tables(self):
        """The reference's joint law P(i, j) ~ ||A[I_i, J_j]||_F^2
        (solvers.py:204-229) with its arithmetic: every submatrix weight is
        numpy's `flat @ flat` on the C-order submatrix (scipy `data @ data`
        when sparse), the per-column conditionals are WeightedSamplers over
        the nonzero weights, and the scales alpha / w; the device samples
        with exactly these arrays, so the (j, i) sequence is the reference's."""
        from .sampling import WeightedSampler

        a = self.a
        s, t = len(self.row_partition), len(self.col_partition)
        col_sel = [slice(i.start, i.stop) if isinstance(i, range) else i for i in self.col_partition.blocks]
        weights = np.zeros((s, t))
        for i, ridx in enumerate(self.row_partition.blocks):
            rb = a.block_matrix(a.block("row", ridx))
            for j, csel in enumerate(col_sel):
                sub = rb[:, csel]
                if hasattr(sub, "toarray"):
                    w = float(sub.data @ sub.data) if sub.nnz else 0.0
                else:
                    flat = np.ravel(sub)
                    w = float(flat @ flat)
                weights[i, j] = w
        self.dsbgs_scales = [[float(self.alpha / w) if w > 0.0 else None for w in row] for row in weights]
        conditionals = []
        for j in range(t):
            alive = np.flatnonzero(weights[:, j] > 0.0)
            conditionals.append((WeightedSampler(weights[alive, j]), alive))
        self.dsbgs_conditionals = conditionals
        # flat device layout of the same tables (rebk_cfg.dsbgs_*)
        self._ds_off = np.zeros(t + 1, dtype=np.int64)
        self._ds_off[1:] = np.cumsum([alive.size for _, alive in conditionals])
        self._ds_cum = np.ascontiguousarray(np.concatenate([c.cumulative for c, _ in conditionals]), dtype=np.float64)
        self._ds_total = np.asarray([float(c.total) for c, _ in conditionals], dtype=np.float64)
        self._ds_alive = np.ascontiguousarray(np.concatenate([alive for _, alive in conditionals]), dtype=np.int32)
        sc = np.zeros((s, t))
        for i in range(s):
            for j in range(t):
                v = self.dsbgs_scales[i][j]
                sc[i, j] = 0.0 if v is None else v
        self._ds_scale = np.ascontiguousarray(sc, dtype=np.float64)

    def _resolve_partition(self, p: Partition | None, axis: str, axis_len: int) -> Partition:
        algo = self.algorithm
        if algo in ("rk", "rek"):
            if p is None:
                return singleton_partition(axis_len, axis)
            if not p.is_singleton():
                raise ValueError(f"{algo} uses singleton partitions; got blocks of size > 1")
        elif p is None:
            raise ValueError(f"{algo} needs a {axis} partition")
        if p.axis != axis:
            raise ValueError(f"partition axis {p.axis!r} where {axis!r} expected")
        if p.axis_len != axis_len:
            raise ValueError(f"partition covers {p.axis_len} {axis}s, matrix has {axis_len}")
        return p

    # -- device binding ---------------------------------------------------------

    def _prefetch_device(self, row_p: Partition, col_p: Partition | None) -> None:
        """Overlap the H2D copy of a dense A with the host sampler setup when
        the device layout is already known (contiguous column blocks, or no
        column partition): the copy _bind_device/device_matrix will ask for."""
        if self.a.is_sparse or os.environ.get("REBK_PREFETCH", "1") == "0":
            return
        if col_p is not None and not (isinstance(col_p, Partition) and col_p.is_contiguous_in_order()):
            return
        row_order = None if row_p.is_contiguous_in_order() else row_p.order()
        self.a.prefetch_device(row_order, None)

    def _bind_device(self) -> None:
        self.row_order = None if self.row_partition.is_contiguous_in_order() else self.row_partition.order()
        self.col_order = None
        if self.col_partition is not None and not self.col_partition.is_contiguous_in_order():
            self.col_order = self.col_partition.order()
        self._row_ptr = self.row_partition.pointers()
        self._row_cum = np.ascontiguousarray(self.row_sampler.cumulative, dtype=np.float64)
        self._row_scale = np.asarray(self.row_scales, dtype=np.float64)
        if self.extended or self.algorithm == "dsbgs":
            self._col_ptr = self.col_partition.pointers()
            self._col_cum = np.ascontiguousarray(self.col_sampler.cumulative, dtype=np.float64)
            self._col_scale = np.asarray(self.col_scales, dtype=np.float64)
        self._dev = None

    @property
    def device_matrix(self):
        if self._dev is None:
            self._dev = self.a.device(self.row_order, self.col_order)
        return self._dev

    def make_cfg(self, *, stop_mode: str, tol: float, stride: int, max_iters: int, key=(0, 0),
                 draw_offset: int = 0, picks: np.ndarray | None = None, record: bool = False,
                 residual_scale: float = 1.0, grid_ctas: int = 0) -> _lib.RebkCfg:
        cfg = _lib.RebkCfg()
        cfg.algorithm = _lib.ALGO_CODES[self.algorithm]
        cfg.stop_mode = _lib.STOP_CODES[stop_mode]
        cfg.tol = float(tol)
        cfg.check_stride = int(stride)
        cfg.max_iters = int(max_iters)
        cfg.philox_key[0], cfg.philox_key[1] = int(key[0]), int(key[1])
        cfg.draw_offset = int(draw_offset)
        cfg.n_row_blocks = len(self.row_partition)
        cfg.row_ptr = _lib.i64ptr(self._row_ptr)
        cfg.row_cum = _lib.dptr(self._row_cum)
        cfg.row_total = float(self.row_sampler.total)
        cfg.row_scale = _lib.dptr(self._row_scale)
        if self.extended or self.algorithm == "dsbgs":
            cfg.n_col_blocks = len(self.col_partition)
            cfg.col_ptr = _lib.i64ptr(self._col_ptr)
            cfg.col_cum = _lib.dptr(self._col_cum)
            cfg.col_total = float(self.col_sampler.total)
            cfg.col_scale = _lib.dptr(self._col_scale)
        if self.algorithm == "dsbgs":
            cfg.dsbgs_off = _lib.i64ptr(self._ds_off)
            cfg.dsbgs_cum = _lib.dptr(self._ds_cum)
            cfg.dsbgs_total = _lib.dptr(self._ds_total)
            cfg.dsbgs_alive = self._ds_alive.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            cfg.dsbgs_scale = _lib.dptr(self._ds_scale)
        if picks is not None:
            cfg.picks = picks.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        cfg.record_errors = int(bool(record))
        cfg.grid_ctas = int(grid_ctas)
        cfg.residual_scale = float(residual_scale)
        return cfg

    def _to_dev_rows(self, v):
        return v if (v is None or self.row_order is None) else v[self.row_order]

    def _to_dev_cols(self, v):
        return v if (v is None or self.col_order is None) else v[self.col_order]

    def _from_dev_rows(self, v):
        if v is None or self.row_order is None:
            return v
        out = np.empty_like(v)
        out[self.row_order] = v
        return out

    def _from_dev_cols(self, v):
        if v is None or self.col_order is None:
            return v
        out = np.empty_like(v)
        out[self.col_order] = v
        return out

    def device_run(self, cfg: _lib.RebkCfg, x0: np.ndarray, z0: np.ndarray | None,
                   x_star: np.ndarray | None, errors_cap: int = 0):
        """One rebk_run call with host buffers: returns (x, z, trace)."""
        lib = _lib.load()
        dm = self.device_matrix
        b = np.ascontiguousarray(self._to_dev_rows(self.b), dtype=np.float64)
        x0d = np.ascontiguousarray(self._to_dev_cols(x0), dtype=np.float64)
        z0d = None if z0 is None else np.ascontiguousarray(self._to_dev_rows(z0), dtype=np.float64)
        xsd = None if x_star is None else np.ascontiguousarray(self._to_dev_cols(x_star), dtype=np.float64)
        x_out = np.empty(self.a.cols, dtype=np.float64)
        z_out = np.empty(self.a.rows, dtype=np.float64) if self.extended else None
        tr = _lib.RebkTrace()
        errs = None
        if errors_cap > 0:
            errs = np.zeros(errors_cap, dtype=np.float64)
            tr.errors = _lib.dptr(errs)
            tr.errors_cap = errors_cap
        rc = lib.rebk_run(dm.handle, ctypes.byref(cfg), _lib.dptr(b), _lib.dptr(x0d), _lib.dptr(z0d),
                          _lib.dptr(xsd), _lib.dptr(x_out), _lib.dptr(z_out), ctypes.byref(tr))
        _lib.check(rc, "rebk_run")
        return self._from_dev_cols(x_out), self._from_dev_rows(z_out), tr, errs

    # -- reference per-step API -------------------------------------------------

    def initial_state(self) -> SolverState:
        n, m = self.a.cols, self.a.rows
        if self.config.x0 is None:
            x = np.zeros(n)
        else:
            x = np.array(self.config.x0, dtype=np.float64, copy=True)
            if x.shape != (n,):
                raise ValueError(f"x0 must have length {n}")
            self._check_start_hypotheses(x=x)
        z = None
        if self.extended:
            if self.config.z0 is None:
                z = self.b.copy()
            else:
                z = np.array(self.config.z0, dtype=np.float64, copy=True)
                if z.shape != (m,):
                    raise ValueError(f"z0 must have length {m}")
                self._check_start_hypotheses(z=z)
        return SolverState(x=x, z=z, k=0, rng=Rng(self.config.seed))

    def _check_start_hypotheses(self, x=None, z=None):
        # flagged, not rejected (solvers.py:251-265)
        f = self.problem.oracle
        if f is None:
            return
        if x is not None and np.any(x):
            drift = np.linalg.norm(x - f.v @ (f.v.T @ x))
            if drift > 1e-8 * np.linalg.norm(x):
                self.warnings.append("x0 outside range(A^T): convergence hypotheses not met")
        if z is not None:
            w = z - self.b
            if np.any(w):
                drift = np.linalg.norm(w - f.u @ (f.u.T @ w))
                if drift > 1e-8 * np.linalg.norm(w):
                    self.warnings.append("z0 outside b + range(A): convergence hypotheses not met")

    def draw_picks(self, rng) -> tuple[int, int]:
        """The two draws of one iteration, in the reference's stream layout
        (solvers.py:8-12): column draw first (discarded without a column
        sweep), then the row draw."""
        if self.algorithm == "dsbgs":  # step_dsbgs, solvers.py:373-375
            j = self.col_sampler.sample(rng)
            conditional, alive = self.dsbgs_conditionals[j]
            return j, int(alive[conditional.sample(rng)])
        if self.extended:
            j = self.col_sampler.sample(rng)
        else:
            rng.uniform()
            j = -1
        i = self.row_sampler.sample(rng)
        return j, i

    def step(self, state: SolverState) -> SolverState:
        j, i = self.draw_picks(state.rng)
        picks = np.asarray([j, i], dtype=np.int32)
        cfg = self.make_cfg(stop_mode="max_iters_only", tol=1.0, stride=1, max_iters=1, picks=picks)
        x_new, z_new, _, _ = self.device_run(cfg, state.x, state.z if self.extended else None, None)
        state.x[...] = x_new
        if self.extended:
            state.z[...] = z_new
        state.k += 1
        return state

    def close(self):
        self._dev = None


def prepare(problem: ProblemInstance, config: SolverConfig) -> SolverContext:
    return SolverContext(problem, config)


def _residual_scale(ctx: SolverContext) -> float:
    scale = float(np.sqrt(ctx.a.frobenius_sq()) * np.linalg.norm(ctx.b))
    return 1.0 if scale == 0.0 else scale


def run(problem: ProblemInstance, config: SolverConfig) -> RunTrace:
    """Iterate on the device until the stopping rule fires or max_iters is
    reached (solvers.py:425-474)."""
    ctx = prepare(problem, config)
    state = ctx.initial_state()
    stop = config.stop
    x_star = None
    if stop.mode == "oracle_error":
        if problem.x_star is None:
            raise ValueError("oracle_error stopping needs a problem with x_star")
        x_star = np.asarray(problem.x_star, dtype=np.float64)
    has_error = stop.mode != "max_iters_only"
    record = bool(config.record_errors and has_error)
    cap = (config.max_iters // stop.check_stride + 2) if record else 0
    key = _lib.philox_key(config.seed)
    cfg = ctx.make_cfg(
        stop_mode=stop.mode, tol=stop.tol, stride=stop.check_stride, max_iters=config.max_iters,
        key=key, record=record,
        residual_scale=_residual_scale(ctx) if stop.mode == "residual_proxy" else 1.0,
    )
    x, z, tr, errs = ctx.device_run(cfg, state.x, state.z, x_star, errors_cap=cap)
    errors = checkpoints = None
    if record:
        nc = int(tr.n_checks)
        errors = errs[:nc].copy()
        checkpoints = np.minimum(np.arange(nc, dtype=np.int64) * stop.check_stride, config.max_iters)
    return RunTrace(
        iters=int(tr.iters),
        converged=bool(tr.converged),
        wall_time=float(tr.loop_ms) / 1e3,
        final_error=float(tr.final_error) if (has_error and tr.has_error) else None,
        errors=errors,
        checkpoints=checkpoints,
        warnings=tuple(ctx.warnings),
        x=x,
        z=z,
        grid_ctas=int(tr.grid_ctas),
        nonfinite_at=None if int(tr.nonfinite_at) < 0 else int(tr.nonfinite_at),
        kernel_path=int(tr.kernel_path),
    )


def resume(problem: ProblemInstance, config: SolverConfig, trace: RunTrace) -> RunTrace:
    """Continue a run from the state a RunTrace carries (resume =
    (x, z, k); the reference's SolverState (solvers.py:88-93) is resumable
    in-process only).  `config` is the configuration of the WHOLE run
    (same seed, partitions, stepsize; `max_iters` the total budget): the
    device continues at iteration trace.iters + 1 with the Philox stream
    advanced past the 2 * trace.iters uniforms already consumed, so the
    iterates are the ones an uninterrupted run(problem, config) computes
    (bitwise when both use the same kernel).  The returned trace counts
    iterations from the start of the whole run.

    The checks of the continued run fall on multiples of check_stride
    counted from trace.iters, so trace.iters must be a multiple of
    check_stride (it is whenever the first leg stopped at a check or at a
    budget that is one)."""
    if trace.x is None:
        raise ValueError("resume needs a RunTrace carrying the iterates (x, z)")
    ctx = prepare(problem, config)
    if ctx.extended and trace.z is None:
        raise ValueError("resume of an extended method needs the trace's z")
    stop = config.stop
    k0 = int(trace.iters)
    if k0 < 0 or k0 > config.max_iters:
        raise ValueError("trace.iters lies outside the run's iteration budget")
    if stop.mode != "max_iters_only" and k0 % stop.check_stride != 0:
        raise ValueError("resume needs trace.iters to be a multiple of check_stride")
    x_star = None
    if stop.mode == "oracle_error":
        if problem.x_star is None:
            raise ValueError("oracle_error stopping needs a problem with x_star")
        x_star = np.asarray(problem.x_star, dtype=np.float64)
    x0 = np.asarray(trace.x, dtype=np.float64)
    z0 = np.asarray(trace.z, dtype=np.float64) if ctx.extended else None
    if x0.shape != (ctx.a.cols,) or (z0 is not None and z0.shape != (ctx.a.rows,)):
        raise ValueError("the trace's iterates do not match the problem's shape")
    has_error = stop.mode != "max_iters_only"
    record = bool(config.record_errors and has_error)
    left = config.max_iters - k0
    cap = (left // stop.check_stride + 2) if record else 0
    cfg = ctx.make_cfg(
        stop_mode=stop.mode, tol=stop.tol, stride=stop.check_stride, max_iters=left,
        key=_lib.philox_key(config.seed), draw_offset=2 * k0, record=record,
        residual_scale=_residual_scale(ctx) if stop.mode == "residual_proxy" else 1.0,
    )
    x, z, tr, errs = ctx.device_run(cfg, x0, z0, x_star, errors_cap=cap)
    errors = checkpoints = None
    if record:
        nc = int(tr.n_checks)
        errors = errs[:nc].copy()
        checkpoints = k0 + np.minimum(np.arange(nc, dtype=np.int64) * stop.check_stride, left)
    return RunTrace(
        iters=k0 + int(tr.iters),
        converged=bool(tr.converged),
        wall_time=float(tr.loop_ms) / 1e3,
        final_error=float(tr.final_error) if (has_error and tr.has_error) else None,
        errors=errors,
        checkpoints=checkpoints,
        warnings=tuple(ctx.warnings),
        x=x,
        z=z,
        grid_ctas=int(tr.grid_ctas),
        nonfinite_at=None if int(tr.nonfinite_at) < 0 else k0 + int(tr.nonfinite_at),
        kernel_path=int(tr.kernel_path),
    )


def default_partitions(a: Matrix, tau_row: int, tau_col: int | None = None):
    row = contiguous_partition(a.rows, min(tau_row, a.rows), "row")
    col = contiguous_partition(a.cols, min(tau_col or tau_row, a.cols), "col")
    return row, col


# -- step functions / plugin registry (solvers.py:306-392) ---------------------


def step_rebk(state: SolverState, ctx: SolverContext) -> SolverState:
    """Column-block sweep on z, then row-block sweep on x against b - z."""
    return ctx.step(state)


def step_rek(state: SolverState, ctx: SolverContext) -> SolverState:
    return ctx.step(state)


def step_rabk(state: SolverState, ctx: SolverContext) -> SolverState:
    return ctx.step(state)


def step_rk(state: SolverState, ctx: SolverContext) -> SolverState:
    return ctx.step(state)


def step_dsbgs(state: SolverState, ctx: SolverContext) -> SolverState:
    """Sampled column coordinates updated from the sampled row residuals."""
    return ctx.step(state)


_STEPPERS = {"rk": step_rk, "rek": step_rek, "rabk": step_rabk, "rebk": step_rebk, "dsbgs": step_dsbgs}

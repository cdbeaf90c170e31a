"""Multi-right-hand-side fp32 REBK (BASELINE config 5).

The reference solves one right-hand side per run (b is 1-D,
solvers.py:141-143) in fp64.  Config 5 batches R right-hand sides that share
one seeded block sequence; every column then follows exactly the
single-RHS REBK iteration (solvers.py:324-337), so the batch is R reference
runs done at once, with the four block products as GEMMs (librebk
``rebk_run_mrhs``).

Sampler arrays: the block weights ||A_block||_F^2 of the fp64 upcast of A.
By default they are computed on the device from the fp32 copy the run uses
anyway (squares accumulated in fp64: the reference's weights up to the
rounding of its `flat @ flat` order, ~1e-15, which could move a pick only if a
uniform fell that close to a CDF boundary; tests/test_gpu_parity.py checks
the sequences agree); passing ``a64`` (a host Matrix of the upcast) selects
the reference's own arithmetic on the host instead.  Each column records the
first check at which ||X_c - X*_c|| <= tol_c (that column's ITER) and the run
stops when every column has crossed.
"""

from __future__ import annotations

import ctypes
import os
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .matrix import Matrix
from .problems import ProblemInstance, ProblemMeta
from .sampling import WeightedSampler
from .solvers import SolverConfig, SolverContext

KERNEL_PATHS = {4: "cuBLAS FP32 GEMMs", 5: "cuBLAS FP32 GEMMs emulated on BF16 tensor cores (BF16x9)",
                8: "hand-written tcgen05 kind::tf32 kernels, 3xTF32 (persistent whole-run kernel by default)"}


class DeviceMatrix32:
    """Owning handle of an fp32 dense rebk_ctx."""

    def __init__(self, a32: np.ndarray, device: int = 0):
        lib = _lib.load()
        a = np.ascontiguousarray(a32, dtype=np.float32)
        handle = ctypes.c_void_p()
        rc = lib.rebk_ctx_create_dense_f32(a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), a.shape[0], a.shape[1],
                                           a.shape[1], device, ctypes.byref(handle))
        _lib.check(rc, "rebk_ctx_create_dense_f32")
        self.handle = handle
        self.shape = a.shape

    def block_frobenius_sq(self, axis: int, ptr: np.ndarray) -> np.ndarray:
        """||A_block||_F^2 of contiguous row (axis 0) or column (axis 1)
        blocks, accumulated in fp64 on the device (matrix.py:170-189)."""
        ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        out = np.empty(ptr.size - 1, dtype=np.float64)
        _lib.check(_lib.load().rebk_block_frobenius_sq(self.handle, axis, out.size, _lib.i64ptr(ptr), _lib.dptr(out)),
                   "rebk_block_frobenius_sq")
        return out

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().rebk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class _DeviceWeightsContext:
    """The part of SolverContext a multi-RHS run needs (validation of the
    config as in solvers.py:123-187, partitions, sampler arrays), with the
    block weights taken from the device copy of A instead of a host upcast."""

    make_cfg = SolverContext.make_cfg
    _resolve_partition = SolverContext._resolve_partition

    def __init__(self, dm: DeviceMatrix32, m: int, n: int, config: SolverConfig):
        algo = config.algorithm.lower()
        if algo not in ("rebk", "rek", "rabk", "rk"):
            raise NotImplementedError(f"multi-RHS runs support rebk, rek, rabk and rk; got {config.algorithm!r}")
        if config.alpha <= 0.0:
            raise ValueError("alpha must be positive")
        if config.max_iters < 0:
            raise ValueError("max_iters must be nonnegative")
        self.algorithm = algo
        self.alpha = float(config.alpha)
        self.extended = algo in ("rebk", "rek")
        self.row_partition = self._resolve_partition(config.row_partition, "row", m)
        self.col_partition = None
        if algo in ("rebk", "rek"):
            self.col_partition = self._resolve_partition(config.col_partition, "col", n)
        self.row_order = None if self.row_partition.is_contiguous_in_order() else self.row_partition.order()
        self.col_order = None
        if self.col_partition is not None and not self.col_partition.is_contiguous_in_order():
            self.col_order = self.col_partition.order()
        if self.row_order is not None or self.col_order is not None:
            return  # the caller refuses non-contiguous partitions
        self._row_ptr = self.row_partition.pointers()
        self.row_sampler = _block_sampler(dm.block_frobenius_sq(0, self._row_ptr))
        self._row_cum = np.ascontiguousarray(self.row_sampler.cumulative, dtype=np.float64)
        self._row_scale = np.asarray([float(self.alpha / w) for w in self.row_sampler.weights], dtype=np.float64)
        if self.extended:
            self._col_ptr = self.col_partition.pointers()
            self.col_sampler = _block_sampler(dm.block_frobenius_sq(1, self._col_ptr))
            self._col_cum = np.ascontiguousarray(self.col_sampler.cumulative, dtype=np.float64)
            self._col_scale = np.asarray([float(self.alpha / w) for w in self.col_sampler.weights], dtype=np.float64)


def _block_sampler(weights: np.ndarray) -> WeightedSampler:
    try:
        return WeightedSampler(weights)
    except ValueError as exc:
        raise ValueError(f"invalid block weights: {exc}") from exc


@dataclass
class MultiRhsTrace:
    iters: int                  # iteration at which the last column crossed (or max_iters)
    iters_per_rhs: np.ndarray   # each column's ITER (first crossing; max_iters if never)
    converged: bool
    wall_time: float            # device time of the loop
    errors_at_iters: np.ndarray  # ||X_c - X*_c|| at each column's ITER
    X: np.ndarray
    Z: np.ndarray | None
    kernel_path: int


def run_multi(a32: np.ndarray, B: np.ndarray, config: SolverConfig, X_star: np.ndarray | None = None,
              tols: np.ndarray | None = None, device_matrix: DeviceMatrix32 | None = None,
              a64: Matrix | None = None) -> MultiRhsTrace:
    """REBK on R right-hand sides at once (fp32 storage and arithmetic).

    a32: (m, n) float32; B: (m, R); X_star: (n, R) for oracle_error stopping;
    tols: per-column absolute tolerances (default config.stop.tol for all).
    """
    a32 = np.ascontiguousarray(a32, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    m, n = a32.shape
    if B.ndim != 2 or B.shape[0] != m:
        raise ValueError("right-hand side block must be (m, R)")
    R = B.shape[1]
    dm = device_matrix
    if a64 is not None:
        prob = ProblemInstance(a=a64, b=B[:, 0].astype(np.float64), x_star=None, b_perp=None,
                               meta=ProblemMeta(0, None, False, 0, 0.0))
        ctx = SolverContext(prob, config)  # the reference's validation and sampler arrays
    else:
        if dm is None:
            dm = DeviceMatrix32(a32)
        ctx = _DeviceWeightsContext(dm, m, n, config)
    if ctx.row_order is not None or ctx.col_order is not None:
        raise NotImplementedError("multi-RHS runs need contiguous partitions")
    stop = config.stop
    if stop.mode == "residual_proxy":
        raise NotImplementedError("multi-RHS runs support oracle_error and max_iters_only")
    if stop.mode == "oracle_error" and X_star is None:
        raise ValueError("oracle_error stopping needs a problem with x_star")
    cfg = ctx.make_cfg(stop_mode=stop.mode, tol=stop.tol, stride=stop.check_stride, max_iters=config.max_iters,
                       key=_lib.philox_key(config.seed))
    if dm is None:
        dm = DeviceMatrix32(a32)
    fp = ctypes.POINTER(ctypes.c_float)
    Xs = None if X_star is None else np.ascontiguousarray(X_star, dtype=np.float32)
    tol_arr = np.full(R, float(stop.tol)) if tols is None else np.ascontiguousarray(tols, dtype=np.float64)
    X0 = None if config.x0 is None else np.ascontiguousarray(config.x0, dtype=np.float32)
    Z0 = None if config.z0 is None else np.ascontiguousarray(config.z0, dtype=np.float32)
    X = np.empty((n, R), dtype=np.float32)
    Z = np.empty((m, R), dtype=np.float32) if ctx.extended else None
    iters = np.empty(R, dtype=np.int64)
    errs = np.empty(R, dtype=np.float64)
    tr = _lib.RebkTrace()

    def p(a):
        return None if a is None else a.ctypes.data_as(fp)

    rc = _lib.load().rebk_run_mrhs(dm.handle, ctypes.byref(cfg), R, p(B), p(X0), p(Z0), p(Xs), _lib.dptr(tol_arr),
                                   p(X), p(Z), _lib.i64ptr(iters), _lib.dptr(errs), ctypes.byref(tr))
    _lib.check(rc, "rebk_run_mrhs")
    if int(tr.kernel_path) in (4, 5) and os.environ.get("REBK_MRHS_MATH", "tc") == "tc":
        # not silent: the shape is outside the hand-written tcgen05 kernel's
        # range (m, n divisible by 4, blocks <= 256 wide, <= 64 RHS) and the
        # library ran its cuBLAS SGEMM path instead (trace.kernel_path 4)
        warnings.warn(f"multi-RHS shape {m}x{n} with {R} RHS is outside the tcgen05 kernel's range; ran the cuBLAS "
                      f"SGEMM path ({KERNEL_PATHS[int(tr.kernel_path)]})", RuntimeWarning, stacklevel=2)
    return MultiRhsTrace(iters=int(tr.iters), iters_per_rhs=iters, converged=bool(tr.converged),
                         wall_time=float(tr.loop_ms) / 1e3, errors_at_iters=errs, X=X, Z=Z,
                         kernel_path=int(tr.kernel_path))

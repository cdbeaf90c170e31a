"""Synthetic instances standing in for BASELINE.json's five configurations.

No public dataset is involved: every config is a seeded synthetic recipe with
the shapes and value distributions BASELINE.json names.
All randomness comes from the reference's own stream family (numpy Philox via
:class:`Rng`), so A is bit-identical on every machine; anything that goes
through LAPACK (QR, Cholesky) may differ in the last bits between hosts,
which is why parity tests compare the device with the oracle on the *same*
in-process instance and use the committed golden vectors with a tolerance.

Stepsize: the "reference stepsize rule" alpha = 1/beta_max (cli.py default
``--alpha 1x``, PAPER.md Remark 2.8); beta_max via block Gram eigenvalues.
Stop: ||x - x*|| / ||x*|| < 1e-6 as the reference's absolute oracle_error
with tol = 1e-6 ||x*|| (1e-4 for C5).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .matrix import Matrix
from .problems import ProblemInstance, ProblemMeta
from .sampling import Partition, Rng, contiguous_partition
from .solvers import SolverConfig, StoppingRule, compute_beta_max


@dataclass
class Workload:
    name: str
    problem: ProblemInstance
    row_partition: Partition
    col_partition: Partition
    alpha: float
    beta_max: float
    rel_tol: float
    seed: int = 17

    def config(self, max_iters: int = 50_000, **kw) -> SolverConfig:
        xs = np.asarray(self.problem.x_star)
        tol = self.rel_tol * float(np.linalg.norm(xs))
        stop = kw.pop("stop", StoppingRule(mode="oracle_error", tol=tol, check_stride=1))
        return SolverConfig(
            algorithm=kw.pop("algorithm", "rebk"), alpha=self.alpha,
            row_partition=self.row_partition, col_partition=self.col_partition,
            seed=kw.pop("seed", self.seed), max_iters=max_iters, stop=stop,
            beta_max=self.beta_max, **kw,
        )

    @property
    def algorithmic_bytes_per_iter(self) -> float:
        """8 (m |J| + |I| n): the two selected blocks read once;
        sparse: 12 B per stored entry of the two blocks (value + index)."""
        m, n = self.problem.a.shape
        if self.problem.a.is_sparse:
            nnz = self.problem.a.nnz
            return 12.0 * nnz * (max(self.col_partition.block_sizes()) / n + max(self.row_partition.block_sizes()) / m)
        tj = max(self.col_partition.block_sizes())
        ti = max(self.row_partition.block_sizes())
        return 8.0 * (m * tj + ti * n)


def _instance(a: np.ndarray, b: np.ndarray, x_star: np.ndarray, seed: int, rank: int) -> ProblemInstance:
    mat = Matrix.from_dense(a)
    return ProblemInstance(
        a=mat, b=b, x_star=x_star, b_perp=None,
        meta=ProblemMeta(declared_rank=rank, kappa_bound=None, consistent=False, seed=seed,
                         residual_norm=0.0),
    )


def c1_arrays(seed: int = 0):
    """C1: A = randn(2000, 500); b = A x + r, r ⊥ range(A), ||r|| = 0.1 ||A x||."""
    rng = Rng(seed)
    a = rng.standard_normal((2000, 500))
    xs = rng.standard_normal(500)
    w = rng.standard_normal(2000)
    q, _ = np.linalg.qr(a)
    r = w - q @ (q.T @ w)
    ax = a @ xs
    r *= 0.1 * np.linalg.norm(ax) / np.linalg.norm(r)
    b = ax + r
    x_star = np.linalg.lstsq(a, b, rcond=None)[0]
    return a, b, x_star


def c1_matrix(seed: int = 0) -> np.ndarray:
    """Just C1's A (pure Philox stream: identical bits on every host)."""
    return Rng(seed).standard_normal((2000, 500))


def c2_arrays(seed: int = 0):
    """C2: A = U diag(sigma) V^T, 4000 x 10000, rank 2000, sigma ~ U[1, 10]."""
    rng = Rng(seed)
    u = np.linalg.qr(rng.standard_normal((4000, 2000)))[0]
    v = np.linalg.qr(rng.standard_normal((10000, 2000)))[0]
    sig = 1.0 + 9.0 * rng.uniforms(2000)
    a = (u * sig) @ v.T
    xs = rng.standard_normal(10000)
    w = rng.standard_normal(4000)
    r = w - u @ (u.T @ w)
    ax = a @ xs
    r *= 0.1 * np.linalg.norm(ax) / np.linalg.norm(r)
    b = ax + r
    x_star = v @ ((u.T @ b) / sig)
    return a, b, x_star


def c4_matrix(seed: int = 0):
    """C4's A: scipy.sparse.random(200000, 50000, density 1e-3, N(0,1) values)
    drawn from numpy default_rng(seed); returns (csr, rng)
    with the generator positioned after A so x / w follow the recipe."""
    import scipy.sparse as sparse

    g = np.random.default_rng(seed)
    s = sparse.random(200000, 50000, density=1e-3, format="csr", random_state=g, data_rvs=g.standard_normal)
    if np.any(np.diff(s.indptr) == 0) or np.any(np.bincount(s.indices, minlength=50000) == 0):
        raise RuntimeError("empty row/column in the C4 draw: resampling not implemented for this seed")
    return s, g


def c4_arrays(seed: int = 0):
    """C4: sparse 200000 x 50000 (1e7 nnz); b = A x + r, r = (I - A A+) w
    (via LSQR) scaled to 0.1 ||A x||; x* = LSQR(A, b)."""
    from scipy.sparse.linalg import lsqr

    s, g = c4_matrix(seed)
    xs = g.standard_normal(50000)
    w = g.standard_normal(200000)
    y = lsqr(s, w, atol=1e-15, btol=1e-15, iter_lim=2000)[0]
    r = w - s @ y
    ax = s @ xs
    r *= 0.1 * np.linalg.norm(ax) / np.linalg.norm(r)
    b = ax + r
    x_star = lsqr(s, b, atol=1e-15, btol=1e-15, iter_lim=2000)[0]
    return s, b, x_star


def power_beta(mat, p: Partition, iters: int = 40, seed: int = 0) -> float:
    """max over blocks of sigma_1(block)^2 / ||block||_F^2 by power iteration
    (a cheap stand-in for the reference's rate constants on big sparse
    blocks; only used to pick the stepsize of the synthetic workloads)."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for idx in p.blocks:
        view = mat.block(p.axis, idx)
        blk = view.materialize()
        fro = mat.block_frobenius_sq(view)
        v = rng.standard_normal(blk.shape[1])
        lam = 0.0
        for _ in range(iters):
            w = blk.T @ (blk @ v)
            lam = float(np.linalg.norm(w))
            v = w / lam
        worst = max(worst, lam / fro)
    return worst


def c5_arrays(m: int = 50000, n: int = 5000, nrhs: int = 64, seed: int = 0):
    """C5: A = randn(m, n) stored fp32; R right-hand sides B = A X + Rres with
    each residual column in null(Aᵀ), ||Rres_c|| = 0.1 ||A X_c||; X* = G⁻¹AᵀB
    (normal equations on the fp64 upcast, G = AᵀA well conditioned for a
    tall Gaussian).  Returns (A32, B32, X*) with B in fp32 as stored."""
    rng = Rng(seed)
    a32 = rng.standard_normal((m, n)).astype(np.float32)
    x = rng.standard_normal((n, nrhs))
    w = rng.standard_normal((m, nrhs))
    a = a32.astype(np.float64)
    g = a.T @ a
    c = np.linalg.cholesky(g)

    def gsolve(v):
        return np.linalg.solve(c.T, np.linalg.solve(c, v))

    r = w - a @ gsolve(a.T @ w)
    ax = a @ x
    r *= 0.1 * np.linalg.norm(ax, axis=0) / np.linalg.norm(r, axis=0)
    b32 = (ax + r).astype(np.float32)
    x_star = gsolve(a.T @ b32.astype(np.float64))
    return a32, b32, x_star


def make_workload(name: str, a: np.ndarray, b: np.ndarray, x_star: np.ndarray, tau_row: int,
                  tau_col: int, rel_tol: float = 1e-6, beta_max: float | None = None,
                  alpha_factor: float = 1.0, seed: int = 17) -> Workload:
    prob = _instance(a, b, x_star, 0, min(a.shape))
    rp = contiguous_partition(a.shape[0], tau_row, "row")
    cp = contiguous_partition(a.shape[1], tau_col, "col")
    if beta_max is None:
        beta_max = compute_beta_max(prob.a, rp, cp)[2]
    return Workload(name, prob, rp, cp, alpha_factor / beta_max, beta_max, rel_tol, seed)


def build(name: str, **kw) -> Workload:
    if name == "c1":
        a, b, xs = c1_arrays()
        return make_workload("c1", a, b, xs, 100, 100, **kw)
    if name == "c2":
        a, b, xs = c2_arrays()
        return make_workload("c2", a, b, xs, 200, 200, **kw)
    if name == "c4":
        s, b, xs = c4_arrays()
        mat = Matrix.from_sparse(s)
        rp = contiguous_partition(200000, 2000, "row")
        cp = contiguous_partition(50000, 1000, "col")
        beta = kw.pop("beta_max", None) or max(power_beta(mat, rp), power_beta(mat, cp))
        prob = ProblemInstance(a=mat, b=b, x_star=xs, b_perp=None,
                               meta=ProblemMeta(declared_rank=50000, kappa_bound=None, consistent=False, seed=0,
                                                residual_norm=0.0))
        return Workload("c4", prob, rp, cp, kw.pop("alpha_factor", 1.0) / beta, beta, kw.pop("rel_tol", 1e-6),
                        kw.pop("seed", 17))
    raise KeyError(f"unknown workload {name!r}")


@dataclass
class DeviceWorkload:
    """A dense instance that lives in device memory only (C3: 16 GB).  The
    block weights, cumulative sums and scales are computed on the device and
    handed to the C-ABI in the reference's layout (SolverContext fields)."""

    name: str
    a: "object"  # torch.Tensor (m, n) float64, row-major
    b: "object"
    x_star: "object"
    row_ptr: np.ndarray
    col_ptr: np.ndarray
    row_w: np.ndarray
    col_w: np.ndarray
    alpha: float
    beta_max: float
    rel_tol: float = 1e-6
    seed: int = 17

    @property
    def shape(self):
        return tuple(self.a.shape)

    @property
    def algorithmic_bytes_per_iter(self) -> float:
        m, n = self.shape
        return 8.0 * (m * int(np.diff(self.col_ptr).max()) + int(np.diff(self.row_ptr).max()) * n)

    def cfg(self, stop_mode: str, tol: float, max_iters: int):
        """rebk_cfg with the same fields SolverContext.make_cfg fills."""
        from . import _lib

        c = _lib.RebkCfg()
        c.algorithm = _lib.ALGO_CODES["rebk"]
        c.stop_mode = _lib.STOP_CODES[stop_mode]
        c.tol = float(tol)
        c.check_stride = 1
        c.max_iters = int(max_iters)
        k = _lib.philox_key(self.seed)
        c.philox_key[0], c.philox_key[1] = int(k[0]), int(k[1])
        self._keep = [np.ascontiguousarray(v) for v in (self.row_ptr, np.cumsum(self.row_w), self.alpha / self.row_w,
                                                        self.col_ptr, np.cumsum(self.col_w), self.alpha / self.col_w)]
        rp, rc, rs, cp, cc, cs = self._keep
        c.n_row_blocks = len(rp) - 1
        c.row_ptr, c.row_cum, c.row_total, c.row_scale = _lib.i64ptr(rp), _lib.dptr(rc), float(rc[-1]), _lib.dptr(rs)
        c.n_col_blocks = len(cp) - 1
        c.col_ptr, c.col_cum, c.col_total, c.col_scale = _lib.i64ptr(cp), _lib.dptr(cc), float(cc[-1]), _lib.dptr(cs)
        return c


def c3_device(m: int = 200000, n: int = 10000, tau_row: int = 1000, tau_col: int = 500, seed: int = 0,
              device: int = 0) -> DeviceWorkload:
    """BASELINE config 3 built on the GPU with torch (16 GB does not round-trip
    through the host): A = randn(m, n), x* = randn(n), r = (I - A A†) randn(m)
    scaled to 0.1 ||A x*||, b = A x* + r, x* = A†b by Cholesky of AᵀA.
    Seeded torch Philox stands in for the reference's numpy stream (SURVEY
    §8(d.1) C3 gives the same shapes and distributions; ITER differs from its
    576 by the instance).  beta_max from device Lanczos block spectral norms."""
    import torch

    from .matrix import DeviceMatrix

    dev = torch.device("cuda", device)
    g = torch.Generator(device=dev).manual_seed(seed)
    a = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
    xs = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    w = torch.randn(m, dtype=torch.float64, device=dev, generator=g)
    chol = torch.linalg.cholesky(a.T @ a)
    ax = a @ xs
    r = w - a @ torch.cholesky_solve((a.T @ w)[:, None], chol)[:, 0]
    r *= 0.1 * ax.norm() / r.norm()
    b = ax + r
    x_star = torch.cholesky_solve((a.T @ b)[:, None], chol)[:, 0]
    del chol, ax, r, w
    row_ptr = np.array(list(range(0, m, tau_row)) + [m], dtype=np.int64)
    col_ptr = np.array(list(range(0, n, tau_col)) + [n], dtype=np.int64)
    dm = DeviceMatrix.from_device_pointer(a.data_ptr(), m, n, n, device)
    row_w = dm.block_frobenius_sq(0, row_ptr)
    col_w = dm.block_frobenius_sq(1, col_ptr)
    # block spectral norms by device Lanczos (rebk_beta.cu; 1 s here, the
    # reference's per-block Jacobi SVD would take hours at this size)
    sr, _ = dm.block_sigma1_sq(0, row_ptr)
    sc, _ = dm.block_sigma1_sq(1, col_ptr)
    dm.close()
    beta = max(float(np.max(sr / row_w)), float(np.max(sc / col_w)))
    torch.cuda.synchronize(dev)
    return DeviceWorkload("c3", a, b, x_star, row_ptr, col_ptr, row_w, col_w, 1.0 / beta, beta)

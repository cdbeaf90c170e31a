"""Synthetic systems and the A†b oracle at scale.

Same functions and meaning as the reference's generators
(problems.py:60-127): ``gen_type1`` (rank-r U diag(d) Vᵀ with d uniform in
(1, kappa)), ``gen_type2`` (standard normal), ``make_rhs`` (b = A x_gen plus
an optional residual in null(Aᵀ), x* = A†b, b_perp, metadata).  Every random
number comes from the reference's own stream (``Rng``: numpy Philox over
SeedSequence, drawn in the reference's order), so the inputs of each
factorisation are bit-identical to the reference's.  What moves to the B200
is the dense linear algebra the reference does with a one-sided Jacobi SVD
in Python (factorizations.py:57-138; infeasible beyond ~4k x 10k):

* the QR factors of gen_type1 and the product (U d) Vᵀ: cuSOLVER geqrf /
  orgqr and a cuBLAS GEMM (torch.linalg on the device: library calls, not
  the hot path);
* the oracle: a thin SVD computed as A = QR (tall) or Aᵀ = QR (wide) and an
  SVD of the small triangular factor, truncated with the reference's rank
  rule (sigma > max(m, n) eps sigma_1); then x* = V diag(1/sigma) Uᵀ b and
  b_perp = b - U Uᵀ b exactly as pinv_apply / residual_split
  (factorizations.py:141-155).

Numerically this is the same oracle through a different (Householder) SVD
algorithm: x*, b_perp agree with the reference's within ~1e-13 relative on
well-conditioned instances (tests/test_generators.py against the
reference's own outputs), and the numerical rank is the same.

``device`` defaults to the first CUDA device; ``device="cpu"`` runs the same
torch code on the host (used by the CPU tests; slow at scale).
"""

from __future__ import annotations

import numpy as np

from .matrix import Matrix
from .problems import ProblemInstance, ProblemMeta, Svd
from .sampling import Rng

CONSISTENCY_RTOL = 1e-8  # problems.py:23
_EPS = float(np.finfo(np.float64).eps)


def _torch_device(device):
    import torch

    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("generators run on a CUDA device (pass device='cpu' for the host torch path)")
        return torch.device("cuda", 0)
    return torch.device(device)


def _qr_q(x, dev):
    import torch

    return torch.linalg.qr(torch.from_numpy(np.ascontiguousarray(x)).to(dev), mode="reduced")[0]


def gen_type1(m: int, n: int, r: int, kappa: float, seed: int, device=None) -> Matrix:
    """Rank-r U D Vᵀ with singular values uniform in (1, kappa) (problems.py:60-74)."""
    if m < 1 or n < 1 or not 1 <= r <= min(m, n):
        raise ValueError(f"need 1 <= r <= min(m, n); got m={m}, n={n}, r={r}")
    if not kappa > 1.0:
        raise ValueError(f"kappa must exceed 1, got {kappa}")
    dev = _torch_device(device)
    rng = Rng(seed)
    u = _qr_q(rng.standard_normal((m, r)), dev)
    v = _qr_q(rng.standard_normal((n, r)), dev)
    import torch

    d = torch.from_numpy(1.0 + (kappa - 1.0) * rng.uniforms(r)).to(dev)
    a = (u * d) @ v.T
    return Matrix.from_dense(a.cpu().numpy())


def gen_type2(m: int, n: int, seed: int) -> Matrix:
    """Standard normal A (problems.py:77-81): the reference's stream itself."""
    if m < 1 or n < 1:
        raise ValueError(f"matrix shape must be positive, got {m}x{n}")
    return Matrix.from_dense(Rng(seed).standard_normal((m, n)))


def device_svd(a, device=None, keep_on_device: bool = False) -> Svd:
    """Thin SVD truncated at rank_tol = max(m, n) eps sigma_1 (the
    reference's svd(), factorizations.py:109-138), on the device: QR of the
    tall orientation, SVD of the small triangular factor."""
    import torch

    dev = _torch_device(device)
    if isinstance(a, Matrix):
        dense = a.to_dense() if not a.is_sparse else a._csr.toarray()
        t = torch.from_numpy(np.ascontiguousarray(dense)).to(dev)
    elif isinstance(a, torch.Tensor):
        t = a.to(dev, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    if t.ndim != 2 or t.numel() == 0:
        raise ValueError("svd needs a nonempty 2-D matrix")
    if not bool(torch.isfinite(t).all()):
        raise ValueError("svd needs finite entries")
    if not bool((t != 0).any()):
        raise ValueError("svd of the zero matrix is not defined here")
    m, n = t.shape
    wide = m < n
    w = t.T if wide else t
    q, rr = torch.linalg.qr(w, mode="reduced")
    # cuSOLVER gesvd (QR iteration) on the device: the default driver
    # selection may pick the approximate Jacobi variant, whose vectors are
    # orthonormal only to its stopping tolerance
    kw = {"driver": "gesvd"} if rr.is_cuda else {}
    ur, s, vh = torch.linalg.svd(rr, full_matrices=False, **kw)
    left = q @ ur          # left singular vectors of w
    right = vh.T
    tol = max(m, n) * _EPS * float(s[0])
    keep = s > tol
    left, s, right = left[:, keep], s[keep], right[:, keep]
    u, v = (right, left) if wide else (left, right)
    if keep_on_device:
        return Svd(u=u, sigma=s, v=v, rank_tol=tol)
    return Svd(u=u.cpu().numpy(), sigma=s.cpu().numpy(), v=v.cpu().numpy(), rank_tol=tol)


def numerical_rank(f: Svd) -> int:
    return int((f.sigma > f.rank_tol).sum())


def make_rhs(a: Matrix, seed: int, inconsistent: bool = False, perp_scale: float = 1.0,
             kappa_bound: float | None = None, oracle: Svd | None = None, device=None) -> ProblemInstance:
    """b = A x_gen (+ perp_scale times the null(Aᵀ) part of a fresh normal
    vector), with x* = A†b and b_perp from the device oracle (problems.py:84-127)."""
    f = oracle if oracle is not None else device_svd(a, device)
    rank = numerical_rank(f)
    rng = Rng(seed)
    x_gen = rng.standard_normal(a.cols)
    b = a.matvec(x_gen)
    residual_norm = 0.0
    if inconsistent:
        if rank >= a.rows:
            raise ValueError("no residual possible: A has full row rank, so null(A^T) is trivial")
        w = rng.standard_normal(a.rows)
        r = perp_scale * (w - f.u @ (f.u.T @ w))
        residual_norm = float(np.linalg.norm(r))
        b = b + r
    x_star = f.v @ ((f.u.T @ b) / f.sigma)
    b_perp = b - f.u @ (f.u.T @ b)
    consistent = float(np.linalg.norm(b_perp)) <= CONSISTENCY_RTOL * float(np.linalg.norm(b))
    meta = ProblemMeta(declared_rank=rank, kappa_bound=kappa_bound, consistent=consistent, seed=int(seed),
                       residual_norm=residual_norm)
    return ProblemInstance(a=a, b=b, x_star=x_star, b_perp=b_perp, meta=meta, oracle=f)

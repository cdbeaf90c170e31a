"""Problem containers (problems.py:26-59 of the reference).

The data types the solver entry point consumes.  The generators and the
oracle at scale live in :mod:`paper_2001_04179_b200.generators` (device QR /
SVD instead of the reference's Python Jacobi SVD).  ``ensure_oracle``
completes a ProblemInstance built without ground truth: device SVD when a
CUDA device is present, LAPACK's on the host otherwise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .matrix import Matrix


@dataclass(frozen=True)
class Svd:
    """Thin SVD truncated at numerical rank (factorizations.py:26-37)."""

    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    rank_tol: float

    @property
    def rank(self) -> int:
        return self.sigma.size


def thin_svd(a: Matrix | np.ndarray) -> Svd:
    """LAPACK thin SVD truncated at max(m, n) * eps * sigma_1 (the
    reference's rank rule, factorizations.py:109-138)."""
    d = a.to_dense() if isinstance(a, Matrix) else np.asarray(a, dtype=np.float64)
    u, s, vt = np.linalg.svd(d, full_matrices=False)
    tol = max(d.shape) * float(np.finfo(np.float64).eps) * float(s[0])
    keep = s > tol
    return Svd(u=u[:, keep], sigma=s[keep], v=vt[keep].T, rank_tol=tol)


@dataclass
class ProblemMeta:
    declared_rank: int
    kappa_bound: float | None
    consistent: bool
    seed: int
    residual_norm: float


@dataclass
class ProblemInstance:
    """(A, b) with the oracle ground truth x_star = A^+ b and b_perp."""

    a: Matrix
    b: np.ndarray
    x_star: np.ndarray | None
    b_perp: np.ndarray | None
    meta: ProblemMeta
    oracle: Svd | None = None

    def ensure_oracle(self) -> Svd:
        if self.oracle is None:
            try:
                import torch

                cuda = torch.cuda.is_available()
            except Exception:  # pragma: no cover
                cuda = False
            if cuda:
                from .generators import device_svd

                self.oracle = device_svd(self.a)
            else:
                self.oracle = thin_svd(self.a)
        f = self.oracle
        if self.x_star is None:
            self.x_star = f.v @ ((f.u.T @ self.b) / f.sigma)
        if self.b_perp is None:
            self.b_perp = self.b - f.u @ (f.u.T @ self.b)
        return f

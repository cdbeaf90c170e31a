"""Convergence-rate constants of REBK (the paper's Theorem 2.7 / Remark 2.8
quantities, reference rates.py:20-147) with their expensive parts on the
B200: the per-block spectral norms through device Lanczos
(``device_beta_max``, rebk_beta.cu) and sigma_1 / sigma_r of A through the
device thin SVD (``generators.device_svd``), instead of the reference's
Python Jacobi SVD of every block and of A.

Formulas (F2 = ||A||_F^2, sigma_r the smallest positive singular value):
  delta  = max(|1 - alpha sigma_1^2 / F2|, |1 - alpha sigma_r^2 / F2|)
  eta    = 1 - (2 alpha - alpha^2 beta_rows) sigma_r^2 / F2
  rho    = 1 - (2 alpha - alpha^2 beta_cols) sigma_r^2 / F2,  rho_hat = max(eta, rho)
  alpha* = 2 F2 / (sigma_1^2 + sigma_r^2),  delta* = (sigma_1^2 - sigma_r^2) / (sigma_1^2 + sigma_r^2)
  guaranteed: alpha < 2 / beta_max
"""

from __future__ import annotations

from dataclasses import dataclass

from .matrix import Matrix
from .problems import Svd
from .sampling import Partition


@dataclass(frozen=True)
class RateConstants:
    sigma1_sq: float
    sigma_r_sq: float
    fro_sq: float
    beta_max_rows: float
    beta_max_cols: float
    beta_max: float
    alpha: float
    delta: float
    eta: float
    rho: float
    rho_hat: float
    guaranteed: bool


def compute_delta(f: Svd, fro_sq: float, alpha: float) -> float:
    if alpha <= 0.0:
        raise ValueError(f"alpha must be positive, got {alpha}")
    s1, sr = float(f.sigma[0]) ** 2, float(f.sigma[-1]) ** 2
    return max(abs(1.0 - alpha * s1 / fro_sq), abs(1.0 - alpha * sr / fro_sq))


def optimal_alpha(f: Svd, fro_sq: float) -> tuple[float, float]:
    s1, sr = float(f.sigma[0]) ** 2, float(f.sigma[-1]) ** 2
    return 2.0 * fro_sq / (s1 + sr), (s1 - sr) / (s1 + sr)


def compute_eta_rho(beta_rows: float, beta_cols: float, sigma_r_sq: float, fro_sq: float,
                    alpha: float) -> tuple[float, float, float]:
    if alpha <= 0.0:
        raise ValueError(f"alpha must be positive, got {alpha}")
    eta = 1.0 - (2.0 * alpha - alpha * alpha * beta_rows) * sigma_r_sq / fro_sq
    rho = 1.0 - (2.0 * alpha - alpha * alpha * beta_cols) * sigma_r_sq / fro_sq
    return eta, rho, max(eta, rho)


def beta_max(a: Matrix, row_p: Partition, col_p: Partition) -> tuple[float, float, float]:
    """(beta over row blocks, beta over column blocks, max): device Lanczos
    for dense A, the host eigensolver for sparse A."""
    from .solvers import device_beta_max

    return device_beta_max(a, row_p, col_p)


def rate_constants(a: Matrix, row_p: Partition, col_p: Partition, alpha: float,
                   oracle: Svd | None = None) -> RateConstants:
    from .generators import device_svd

    f = oracle if oracle is not None else device_svd(a)
    fro_sq = a.frobenius_sq()
    br, bc, bm = beta_max(a, row_p, col_p)
    delta = compute_delta(f, fro_sq, alpha)
    sr = float(f.sigma[-1]) ** 2
    eta, rho, rho_hat = compute_eta_rho(br, bc, sr, fro_sq, alpha)
    return RateConstants(sigma1_sq=float(f.sigma[0]) ** 2, sigma_r_sq=sr, fro_sq=fro_sq, beta_max_rows=br,
                         beta_max_cols=bc, beta_max=bm, alpha=alpha, delta=delta, eta=eta, rho=rho, rho_hat=rho_hat,
                         guaranteed=alpha < 2.0 / bm)

"""Generators and the A†b oracle (paper_2001_04179_b200.generators, SURVEY
§8f #2) against the reference's own outputs (tests/golden/generators.npz,
made by tests/golden/gen_generators.py with the reference's Jacobi SVD):
type-1 / type-2 matrices, b, x*, b_perp, rank, consistency and residual
norm.  The random streams are the reference's, so gen_type2 is bit-exact;
the factorisations go through Householder QR/SVD instead of Jacobi, so the
rest agrees to rounding (1e-12 relative).  The CPU tests run the same torch
code on the host; the gpu test repeats them on the B200 and adds an
instance far beyond the reference's Jacobi range."""

import os

import numpy as np
import pytest

from paper_2001_04179_b200 import generators as GN

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "generators.npz"))
CASES = [("t1_tall", 1, (60, 25, 20, 3.0), 11, 12, True, 1.0),
         ("t1_wide", 1, (30, 70, 18, 10.0), 13, 14, True, 0.5),
         ("t1_consistent", 1, (40, 30, 30, 2.0), 15, 16, False, 1.0),
         ("t2_tall", 2, (80, 35), 17, 18, True, 2.0),
         ("t2_wide", 2, (25, 50), 19, 20, False, 1.0)]
RTOL = 1e-12


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def check_case(case, device):
    name, kind, shape, ms, rs, inc, ps = case
    a = GN.gen_type1(*shape, seed=ms, device=device) if kind == 1 else GN.gen_type2(*shape, seed=ms)
    if kind == 2:
        assert np.array_equal(a.to_dense(), G[f"{name}__a"])  # the reference's stream, bit for bit
    else:
        assert rel(a.to_dense(), G[f"{name}__a"]) <= RTOL
    p = GN.make_rhs(a, seed=rs, inconsistent=inc, perp_scale=ps, kappa_bound=shape[3] if kind == 1 else None,
                    device=device)
    rank, consistent, rnorm = G[f"{name}__meta"]
    assert p.meta.declared_rank == int(rank) and p.meta.consistent == bool(consistent)
    assert p.meta.residual_norm == pytest.approx(float(rnorm), rel=RTOL, abs=1e-300)
    assert rel(p.b, G[f"{name}__b"]) <= RTOL
    assert rel(p.x_star, G[f"{name}__x_star"]) <= RTOL
    bp = G[f"{name}__b_perp"]
    assert np.linalg.norm(p.b_perp - bp) <= RTOL * max(np.linalg.norm(p.b), 1.0)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_generators_match_reference_on_host(case):
    check_case(case, "cpu")


def test_full_row_rank_inconsistent_raises():
    a = GN.gen_type2(20, 30, seed=3)
    with pytest.raises(ValueError) as info:
        GN.make_rhs(a, seed=4, inconsistent=True, device="cpu")
    assert str(info.value) == str(G["err_full_row_rank"])


def test_argument_validation():
    with pytest.raises(ValueError, match="need 1 <= r"):
        GN.gen_type1(10, 5, 6, 2.0, seed=0, device="cpu")
    with pytest.raises(ValueError, match="kappa must exceed 1"):
        GN.gen_type1(10, 5, 3, 1.0, seed=0, device="cpu")
    with pytest.raises(ValueError, match="shape must be positive"):
        GN.gen_type2(0, 5, seed=0)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_generators_match_reference_on_device(case):
    check_case(case, None)


@pytest.mark.gpu
def test_oracle_at_scale_on_device():
    """A type-1 instance of 20000 x 4000 (rank 3000), whose Jacobi-SVD oracle
    the reference cannot afford: the device oracle's x* solves the normal
    equations restricted to range(Aᵀ) and b_perp is orthogonal to range(A)."""
    import torch

    a = GN.gen_type1(20000, 4000, 3000, 5.0, seed=1)
    p = GN.make_rhs(a, seed=2, inconsistent=True, perp_scale=0.1)
    assert p.meta.declared_rank == 3000 and not p.meta.consistent
    A = torch.from_numpy(a.to_dense()).cuda()
    xs = torch.from_numpy(p.x_star).cuda()
    b = torch.from_numpy(p.b).cuda()
    bp = torch.from_numpy(p.b_perp).cuda()
    r = b - A @ xs
    assert float(torch.linalg.norm(r - bp) / torch.linalg.norm(b)) <= 1e-10      # A x* = b - b_perp
    assert float(torch.linalg.norm(A.T @ bp) / torch.linalg.norm(b)) <= 1e-10    # b_perp in null(Aᵀ)
    v = torch.from_numpy(p.oracle.v).cuda()
    proj = float(torch.linalg.norm(xs - v @ (v.T @ xs)) / torch.linalg.norm(xs))
    orth = float(torch.linalg.norm(v.T @ v - torch.eye(v.shape[1], dtype=v.dtype, device=v.device)))
    assert proj <= 1e-12 and orth <= 1e-11, (proj, orth)  # x* in range(Aᵀ), V orthonormal

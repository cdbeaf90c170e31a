"""Device block spectral norms: beta_max from Lanczos on the
B200 (rebk_beta.cu) against the reference's own beta (Jacobi SVD,
rates.py:76-90), as recorded in the golden files, and against the host
eigensolver where the reference value is not stored.

beta only enters run() through the OutOfRegimeWarning (solvers.py:180-185)
and the CLI's x-suffixed stepsizes (cli.py:288-302, alpha = factor/beta), so
the bar is the rounding of two different eigensolvers: 1e-12 relative.
"""

import os

import numpy as np
import pytest

import paper_2001_04179_b200 as P
from paper_2001_04179_b200 import _lib

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
BETA_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    assert _lib.device_count() > 0, "gpu tests need a CUDA device (no CPU fallback exists)"


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=True)


def partitions(g, a):
    rp = P.Partition("row", a.shape[0], tuple(np.asarray(b, dtype=np.int64) for b in g["row_blocks"]))
    cp = P.Partition("col", a.shape[1], tuple(np.asarray(b, dtype=np.int64) for b in g["col_blocks"]))
    return rp, cp


# (case, stepsize factor the generator used: alpha = factor / beta_ref), gen_golden.py:156-194
FACTOR_CASES = [("case_t1_40x20_rebk.npz", 1.0), ("case_t2_37x23_ragged.npz", 1.5), ("case_t1_30x50_rebk.npz", 1.75)]


@pytest.mark.parametrize("case,factor", FACTOR_CASES)
def test_device_beta_matches_reference_small_cases(case, factor):
    g = load(case)
    a = g["a"]
    rp, cp = partitions(g, a)
    beta_ref = factor / float(g["alpha"])
    br, bc, bmax = P.device_beta_max(P.Matrix.from_dense(a), rp, cp)
    assert bmax == pytest.approx(beta_ref, rel=BETA_RTOL)
    hr, hc, _ = P.compute_beta_max(P.Matrix.from_dense(a), rp, cp)
    assert br == pytest.approx(hr, rel=BETA_RTOL) and bc == pytest.approx(hc, rel=BETA_RTOL)


def test_device_beta_noncontiguous_partitions():
    g = load("case_t2_20x12_noncontig.npz")
    a = g["a"]
    rp, cp = partitions(g, a)
    assert not rp.is_contiguous_in_order()
    d = P.device_beta_max(P.Matrix.from_dense(a), rp, cp)
    h = P.compute_beta_max(P.Matrix.from_dense(a), rp, cp)
    for x, y in zip(d, h):
        assert x == pytest.approx(y, rel=BETA_RTOL)


def test_device_beta_singleton_and_mixed_blocks():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((30, 17))
    rp = P.Partition("row", 30, (np.arange(0, 1), np.arange(1, 13), np.arange(13, 30)))
    cp = P.singleton_partition(17, "col")
    br, bc, _ = P.device_beta_max(P.Matrix.from_dense(a), rp, cp)
    hr, hc, _ = P.compute_beta_max(P.Matrix.from_dense(a), rp, cp)
    assert bc == 1.0 == hc
    assert br == pytest.approx(hr, rel=BETA_RTOL)


def test_device_beta_c1_matches_reference_jacobi():
    from paper_2001_04179_b200.workloads import c1_matrix

    g = load("c1_golden.npz")
    a = c1_matrix()
    rp, cp = P.contiguous_partition(2000, 100, "row"), P.contiguous_partition(500, 100, "col")
    _, _, bmax = P.device_beta_max(P.Matrix.from_dense(a), rp, cp)
    assert bmax == pytest.approx(float(g["beta"]), rel=BETA_RTOL)


def test_device_beta_c2_matches_reference_jacobi():
    """C2 (4000 x 10000, blocks of 200) against the reference's OWN beta:
    rates.compute_beta_max (one-sided Jacobi SVD of all 70 blocks, 886 s on
    the build host; tests/golden/gen_golden.py --c2-beta)."""
    from paper_2001_04179_b200 import workloads

    ref = load("c2_beta_ref.npz")
    wl = workloads.build("c2", beta_max=1.0)
    br, bc, bmax = P.device_beta_max(wl.problem.a, wl.row_partition, wl.col_partition)
    assert br == pytest.approx(float(ref["beta_rows"]), rel=BETA_RTOL)
    assert bc == pytest.approx(float(ref["beta_cols"]), rel=BETA_RTOL)
    assert bmax == pytest.approx(float(ref["beta"]), rel=BETA_RTOL)
    # the C2 golden run's alpha came from the host Gram eigensolver: same beta
    assert float(load("c2_golden.npz")["beta"]) == pytest.approx(float(ref["beta"]), rel=BETA_RTOL)


def test_prepare_resolves_beta_on_device_and_warns_like_host(monkeypatch):
    g = load("case_t1_40x20_rebk.npz")
    a = g["a"]
    rp, cp = partitions(g, a)
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    beta_ref = 1.0 / float(g["alpha"])
    for factor, warned in ((1.0, False), (2.5, True)):
        cfg = P.SolverConfig(algorithm="rebk", alpha=factor / beta_ref, row_partition=rp, col_partition=cp, seed=9)
        monkeypatch.setenv("REBK_BETA_BACKEND", "device")
        ctx = P.prepare(prob, cfg)
        assert ctx.beta_max == pytest.approx(beta_ref, rel=BETA_RTOL)
        assert (P.OutOfRegimeWarning in ctx.warnings) is warned
        monkeypatch.setenv("REBK_BETA_BACKEND", "host")
        assert P.prepare(prob, cfg).warnings == ctx.warnings


def test_lanczos_steps_bounded_and_deterministic():
    from paper_2001_04179_b200.workloads import c1_matrix

    a = c1_matrix()
    mat = P.Matrix.from_dense(a)
    dm = mat.device()
    ptr = P.contiguous_partition(2000, 100, "row").pointers()
    s1, k1 = dm.block_sigma1_sq(0, ptr)
    s2, k2 = dm.block_sigma1_sq(0, ptr)
    assert np.array_equal(s1, s2) and np.array_equal(k1, k2)
    assert np.all(k1 >= 3) and np.all(k1 <= 100)
    # Ritz values grow monotonically towards sigma_1^2: a 5-step budget stops below
    s5, k5 = dm.block_sigma1_sq(0, ptr, max_steps=5)
    assert np.all(k5 == 5) and np.all(s5 <= s1 * (1 + 1e-14))

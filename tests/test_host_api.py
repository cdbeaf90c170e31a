"""Host-side mirror of the reference interface: validation errors and
setup arrays match the reference (solvers.py:126-202, sampling.py); no
GPU needed because no iteration runs."""

import numpy as np
import pytest

import paper_2001_04179_b200 as P
from paper_2001_04179_b200 import _lib


def problem(m=15, n=8, seed=24):
    a = np.random.default_rng(seed).standard_normal((m, n))
    x = np.random.default_rng(seed + 1).standard_normal(n)
    b = a @ x
    return P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=x, b_perp=None,
                             meta=P.ProblemMeta(n, None, True, seed, 0.0))


def test_unknown_algorithm():
    with pytest.raises(ValueError, match="unknown algorithm"):
        P.prepare(problem(), P.SolverConfig(algorithm="sor"))


def test_alpha_positive():
    with pytest.raises(ValueError, match="alpha must be positive"):
        P.prepare(problem(), P.SolverConfig(algorithm="rek", alpha=0.0))


def test_partition_requirements():
    p = problem()
    with pytest.raises(ValueError, match="partition"):
        P.prepare(p, P.SolverConfig(algorithm="rebk", alpha=1.0))
    with pytest.raises(ValueError, match="partition"):
        P.prepare(p, P.SolverConfig(algorithm="rabk", alpha=1.0))


def test_rek_rejects_non_singleton():
    cfg = P.SolverConfig(algorithm="rek", row_partition=P.contiguous_partition(15, 3, "row"))
    with pytest.raises(ValueError, match="singleton"):
        P.prepare(problem(), cfg)


def test_projection_stepsize_rejected_before_not_implemented():
    cfg = P.SolverConfig(algorithm="rbk", alpha=1.5, row_partition=P.contiguous_partition(15, 3, "row"))
    with pytest.raises(ValueError, match="stepsize"):
        P.prepare(problem(), cfg)
    cfg = P.SolverConfig(algorithm="rbk", alpha=1.0, row_partition=P.contiguous_partition(15, 3, "row"))
    with pytest.raises(NotImplementedError):
        P.prepare(problem(), cfg)


def test_partition_axis_and_length_checks():
    p = problem()
    with pytest.raises(ValueError, match="axis"):
        P.prepare(p, P.SolverConfig(algorithm="rabk", row_partition=P.contiguous_partition(15, 3, "col")))
    with pytest.raises(ValueError, match="covers"):
        P.prepare(p, P.SolverConfig(algorithm="rabk", row_partition=P.contiguous_partition(14, 3, "row")))


def test_rhs_length():
    p = problem()
    p.b = np.ones(3)
    with pytest.raises(ValueError, match="right-hand side"):
        P.prepare(p, P.SolverConfig(algorithm="rek"))


def test_stopping_rule_validation():
    with pytest.raises(ValueError):
        P.StoppingRule(mode="bogus")
    with pytest.raises(ValueError):
        P.StoppingRule(tol=0.0)
    with pytest.raises(ValueError):
        P.StoppingRule(check_stride=0)


def test_sampler_arrays_are_the_reference_ones():
    p = problem(40, 20)
    rp, cp = P.contiguous_partition(40, 5, "row"), P.contiguous_partition(20, 5, "col")
    ctx = P.prepare(p, P.SolverConfig(algorithm="rebk", alpha=1.3, row_partition=rp, col_partition=cp))
    a = p.a.to_dense()
    w = [float(np.ravel(a[i:i + 5]) @ np.ravel(a[i:i + 5])) for i in range(0, 40, 5)]
    assert np.array_equal(ctx.row_sampler.cumulative, np.cumsum(w))
    assert ctx.row_scales == [float(1.3 / v) for v in w]
    cfg = ctx.make_cfg(stop_mode="oracle_error", tol=1e-6, stride=1, max_iters=10, key=_lib.philox_key(3))
    assert cfg.n_row_blocks == 8 and cfg.n_col_blocks == 4
    assert cfg.row_total == ctx.row_sampler.total


def test_noncontiguous_partition_permutation_roundtrip():
    p = problem(12, 6)
    rp = P.Partition("row", 12, (np.array([0, 5, 7]), np.array([1, 2, 3, 4]), np.array([6, 8, 9, 10, 11])))
    cp = P.Partition("col", 6, (np.array([5, 0]), np.array([1, 2, 3, 4])))
    ctx = P.prepare(p, P.SolverConfig(algorithm="rebk", alpha=1.0, row_partition=rp, col_partition=cp))
    assert ctx.row_order is not None and ctx.col_order is not None
    v = np.arange(12.0)
    assert np.array_equal(ctx._from_dev_rows(ctx._to_dev_rows(v)), v)
    w = np.arange(6.0)
    assert np.array_equal(ctx._from_dev_cols(ctx._to_dev_cols(w)), w)
    assert ctx._row_ptr.tolist() == [0, 3, 7, 12]


def test_out_of_regime_warning_without_device():
    p = problem()
    rp, cp = P.contiguous_partition(15, 3, "row"), P.contiguous_partition(8, 2, "col")
    beta = P.compute_beta_max(p.a, rp, cp)[2]
    ctx = P.prepare(p, P.SolverConfig(algorithm="rebk", alpha=2.05 / beta, row_partition=rp, col_partition=cp))
    assert P.OutOfRegimeWarning in ctx.warnings


@pytest.mark.skipif(_lib.device_count() > 0, reason="checks the no-GPU behaviour")
def test_run_without_gpu_raises_not_falls_back():
    with pytest.raises(_lib.RebkError):
        P.run(problem(), P.SolverConfig(algorithm="rek", max_iters=5))


@pytest.mark.parametrize("shape,tau", [((300, 250), 40), ((64, 1000), 200), ((7, 9), 2)])
def test_gathered_column_weights_bitwise(shape, tau):
    """The threaded single-pass column-block gather (rebk_host_gather_col_blocks)
    gives the exact bits of the reference's `flat @ flat` on np.ravel(A[:, J])
    (matrix.py:170-189), ragged last block included."""
    a = np.random.default_rng(5).standard_normal(shape)
    m = P.Matrix.from_dense(a)
    p = P.contiguous_partition(shape[1], tau, "col")
    want = []
    for blk in p.blocks:
        flat = np.ravel(a[:, blk.start:blk.stop])
        want.append(float(flat @ flat))
    got = m.col_block_weights(p.pointers())
    assert got == want
    assert list(P.build_sampler(m, p).weights) == want
    # a partition the gather does not cover keeps the per-block path
    assert m.col_block_weights(np.array([0, shape[1]], dtype=np.int64)) == [float(np.ravel(a) @ np.ravel(a))]


def test_gather_rejects_bad_pointers():
    lib = _lib.load()
    a = np.zeros((4, 6))
    out = np.empty(a.size)
    bad = np.array([0, 3, 3, 6], dtype=np.int64)
    assert lib.rebk_host_gather_col_blocks(_lib.dptr(a), 4, 6, 6, 3, _lib.i64ptr(bad), _lib.dptr(out), 2) != 0


DSBGS_CASES = ["case_t2_37x23_dsbgs.npz", "case_t2_30x20_dsbgs_zero_sub.npz", "case_t2_20x12_dsbgs_noncontig.npz",
               "case_sp_80x40_dsbgs.npz"]


@pytest.mark.parametrize("case", DSBGS_CASES)
def test_dsbgs_joint_sampler_tables_and_picks_match_reference(case):
    """step_dsbgs's joint sampler (solvers.py:204-229): the submatrix scales
    the device consumes and the host pick sequence (column draw, then the
    column's conditional over nonzero row blocks) equal the reference's."""
    import os

    import scipy.sparse as sp

    gold = os.path.join(os.path.dirname(__file__), "golden")
    g = np.load(os.path.join(gold, case), allow_pickle=True)
    if "a_indptr" in g.files:
        a = P.Matrix.from_sparse(sp.csr_matrix((g["a_data"], g["a_indices"], g["a_indptr"]),
                                               shape=tuple(g["a_shape"])))
    else:
        a = P.Matrix.from_dense(g["a"])
    rp = P.Partition("row", a.rows, tuple(np.asarray(b, dtype=np.int64) for b in g["row_blocks"]))
    cp = P.Partition("col", a.cols, tuple(np.asarray(b, dtype=np.int64) for b in g["col_blocks"]))
    prob = P.ProblemInstance(a=a, b=g["b"], x_star=g["x_star"], b_perp=None, meta=P.ProblemMeta(0, None, False, 0, 0.0))
    ctx = P.prepare(prob, P.SolverConfig(algorithm="dsbgs", alpha=float(g["alpha"]), seed=int(g["seed"]),
                                         row_partition=rp, col_partition=cp, max_iters=10))
    got = np.asarray([[np.nan if v is None else v for v in row] for row in ctx.dsbgs_scales])
    np.testing.assert_array_equal(got, g["dsbgs_scales"])
    rng = P.Rng(int(g["seed"]))
    picks = np.asarray([ctx.draw_picks(rng) for _ in range(len(g["picks"]))], dtype=np.int32)
    np.testing.assert_array_equal(picks, g["picks"])
    # the flat device tables describe the same conditionals
    for j, (cond, alive) in enumerate(ctx.dsbgs_conditionals):
        lo, hi = ctx._ds_off[j], ctx._ds_off[j + 1]
        np.testing.assert_array_equal(ctx._ds_cum[lo:hi], cond.cumulative)
        np.testing.assert_array_equal(ctx._ds_alive[lo:hi], alive)


def test_resume_needs_a_trace_with_iterates():
    """resume() refuses a RunTrace without x before touching the device."""
    import pytest

    import paper_2001_04179_b200 as P

    tr = P.RunTrace(iters=10, converged=False, wall_time=0.0, final_error=None)
    with pytest.raises(ValueError, match="iterates"):
        P.resume(None, None, tr)

"""Parity of the B200 path (librebk.so) with the reference, through the
public API and the C ABI.

Gates (BASELINE.json north_star): block-index sequence bit-exact; x, z
within 1e-10 relative (fp64); ITER equal; bitwise run-to-run replay.
Golden vectors come from the reference itself (tests/golden/gen_golden.py);
the oracle restatement checks the same instance in-process.
"""

import ctypes
import glob
import os

import numpy as np
import pytest

import paper_2001_04179_b200 as P
from paper_2001_04179_b200 import _lib
from oracle.rebk_oracle import OracleRng, OracleSolver

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RTOL = 1e-10  # fp64 iterate tolerance stated by the north star


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    assert _lib.device_count() > 0, "gpu tests need a CUDA device (no CPU fallback exists)"


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=True)


def case_problem(g):
    if "a_indptr" in g.files:
        import scipy.sparse as sp

        a = sp.csr_matrix((g["a_data"], g["a_indices"], g["a_indptr"]), shape=tuple(g["a_shape"]))
        mat = P.Matrix.from_sparse(a)
    else:
        a = g["a"]
        mat = P.Matrix.from_dense(a)
    prob = P.ProblemInstance(a=mat, b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    algo = str(g["algorithm"])
    rb = [np.asarray(b, dtype=np.int64) for b in g["row_blocks"]]
    rp = P.Partition("row", a.shape[0], tuple(rb)) if algo not in ("rk", "rek") else None
    cp = None
    if "col_blocks" in g.files and algo not in ("rk", "rek"):
        cp = P.Partition("col", a.shape[1], tuple(np.asarray(b, dtype=np.int64) for b in g["col_blocks"]))
    z0 = g["z0"] if "z0" in g.files else None
    cfg = P.SolverConfig(algorithm=algo, alpha=float(g["alpha"]), row_partition=rp, col_partition=cp,
                         seed=int(g["seed"]), max_iters=int(g["max_iters"]),
                         stop=P.StoppingRule(mode=str(g["mode"]), tol=float(g["tol"]),
                                             check_stride=int(g["stride"])),
                         record_errors=True, z0=z0, beta_max=1e-300)
    return prob, cfg


CASES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLD, "case_*.npz")))


@pytest.mark.parametrize("case", CASES)
def test_run_matches_reference_case(case):
    g = load(case)
    prob, cfg = case_problem(g)
    tr = P.run(prob, cfg)
    assert tr.iters == int(g["iters"])
    assert tr.converged == bool(g["converged"])
    if str(g["mode"]) == "max_iters_only":
        assert tr.final_error is None and tr.errors is None
    else:
        assert tr.final_error == pytest.approx(float(g["final_error"]), rel=1e-9, abs=1e-13)
        assert np.array_equal(tr.checkpoints, g["checkpoints"])
        np.testing.assert_allclose(tr.errors, g["errors"], rtol=1e-9, atol=1e-13)
    k = int(g["iters"])
    if f"x_{k}" in g.files:
        assert rel(tr.x, g[f"x_{k}"]) <= RTOL
        if tr.z is not None:
            assert rel(tr.z, g[f"z_{k}"]) <= RTOL


@pytest.mark.parametrize("case", CASES)
def test_step_snapshots_match_reference_case(case):
    g = load(case)
    prob, cfg = case_problem(g)
    ctx = P.prepare(prob, cfg)
    st = ctx.initial_state()
    ks = set(int(k) for k in g["ks"])
    for k in range(1, max(ks) + 1):
        ctx.step(st)
        if k in ks:
            assert rel(st.x, g[f"x_{k}"]) <= RTOL, k
            if st.z is not None:
                assert rel(st.z, g[f"z_{k}"]) <= RTOL, k


@pytest.mark.parametrize("case", CASES)
def test_device_sampler_sequence_bit_exact(case):
    g = load(case)
    prob, cfg = case_problem(g)
    ctx = P.prepare(prob, cfg)
    want = g["picks"].astype(np.int32)
    c = ctx.make_cfg(stop_mode="max_iters_only", tol=1.0, stride=1, max_iters=len(want),
                     key=_lib.philox_key(int(g["seed"])))
    out = np.empty((len(want), 2), dtype=np.int32)
    rc = _lib.load().rebk_sample_sequence(ctypes.byref(c), 1, len(want),
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    _lib.check(rc, "rebk_sample_sequence")
    assert np.array_equal(out, want)


def test_hand_values_identity():
    # test_solvers.py:307-316
    prob = P.ProblemInstance(a=P.Matrix.from_dense(np.eye(2)), b=np.array([1.0, 2.0]), x_star=None,
                             b_perp=None, meta=P.ProblemMeta(0, None, True, 0, 0.0))
    cfg = P.SolverConfig(algorithm="rebk", alpha=1.0, seed=0, row_partition=P.contiguous_partition(2, 2, "row"),
                         col_partition=P.contiguous_partition(2, 2, "col"), beta_max=1.0)
    ctx = P.prepare(prob, cfg)
    st = ctx.initial_state()
    ctx.step(st)
    assert np.allclose(st.z, [0.5, 1.0], atol=1e-15)
    assert np.allclose(st.x, [0.25, 0.5], atol=1e-15)


class ScriptedRng:
    def __init__(self, values):
        self.values = list(values)

    def uniform(self):
        return self.values.pop(0)


def test_scripted_rek_hand_formula():
    # test_solvers.py:92-109
    rng = np.random.default_rng(1)
    a = rng.standard_normal((5, 3))
    b = rng.standard_normal(5)
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=None, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    ctx = P.prepare(prob, P.SolverConfig(algorithm="rek", seed=0, beta_max=1.0))
    st = ctx.initial_state()
    st.x = rng.standard_normal(3)
    x_before, z_before = st.x.copy(), st.z.copy()
    st.rng = ScriptedRng([0.0, 0.0])
    ctx.step(st)
    col = a[:, 0]
    z_want = z_before - (col @ z_before) / (col @ col) * col
    row = a[0]
    x_want = x_before - (row @ x_before - b[0] + z_want[0]) / (row @ row) * row
    assert np.allclose(st.z, z_want, rtol=1e-13)
    assert np.allclose(st.x, x_want, rtol=1e-13)


def test_scripted_rk_hand_formula():
    # test_solvers.py:75-89
    rng = np.random.default_rng(0)
    a = rng.standard_normal((6, 4))
    b = rng.standard_normal(6)
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=None, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    ctx = P.prepare(prob, P.SolverConfig(algorithm="rk", alpha=0.8, seed=0, beta_max=1.0))
    st = ctx.initial_state()
    st.x = rng.standard_normal(4)
    xb = st.x.copy()
    st.rng = ScriptedRng([0.5, 0.0])
    ctx.step(st)
    row = a[0]
    want = xb - 0.8 * (row @ xb - b[0]) / (row @ row) * row
    assert np.allclose(st.x, want, rtol=1e-13)


def small_problem(m, n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    xs = np.linalg.lstsq(a, b, rcond=None)[0]
    return P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=xs, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, seed, 0.0))


def test_rek_equals_singleton_rebk_bitwise():
    # test_solvers.py:136-151 (bitwise over 1000 steps, via whole runs)
    p = small_problem(12, 7, 2)
    cfg_rek = P.SolverConfig(algorithm="rek", alpha=1.0, seed=17, max_iters=1000,
                             stop=P.StoppingRule(mode="max_iters_only"), beta_max=1.0)
    cfg_rebk = P.SolverConfig(algorithm="rebk", alpha=1.0, seed=17, max_iters=1000,
                              row_partition=P.singleton_partition(12, "row"),
                              col_partition=P.singleton_partition(7, "col"),
                              stop=P.StoppingRule(mode="max_iters_only"), beta_max=1.0)
    t1, t2 = P.run(p, cfg_rek), P.run(p, cfg_rebk)
    assert np.array_equal(t1.x, t2.x) and np.array_equal(t1.z, t2.z)


def test_rebk_zero_z_equals_rabk_bitwise():
    # test_solvers.py:249-265 and :318-329
    p = small_problem(14, 9, 12)
    rp, cp = P.contiguous_partition(14, 3, "row"), P.contiguous_partition(9, 3, "col")
    mk = dict(alpha=1.4, seed=33, max_iters=1000, stop=P.StoppingRule(mode="max_iters_only"), beta_max=1.0)
    t1 = P.run(p, P.SolverConfig(algorithm="rabk", row_partition=rp, **mk))
    t2 = P.run(p, P.SolverConfig(algorithm="rebk", row_partition=rp, col_partition=cp, z0=np.zeros(14), **mk))
    assert not t2.z.any()
    assert np.array_equal(t1.x, t2.x)


def test_replay_determinism_bitwise():
    # test_solvers.py:452-459, on a grid-sized problem so many CTAs reduce
    from paper_2001_04179_b200.workloads import c1_matrix

    g = load("c1_golden.npz")
    prob = P.ProblemInstance(a=P.Matrix.from_dense(c1_matrix()), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    cfg = P.SolverConfig(algorithm="rebk", alpha=1.2 * float(g["alpha"]), seed=7, max_iters=300,
                         row_partition=P.contiguous_partition(2000, 100, "row"),
                         col_partition=P.contiguous_partition(500, 100, "col"),
                         stop=P.StoppingRule(tol=1e-300), beta_max=float(g["beta"]))
    t1, t2 = P.run(prob, cfg), P.run(prob, cfg)
    assert t1.iters == t2.iters
    assert t1.final_error == t2.final_error
    assert np.array_equal(t1.x, t2.x) and np.array_equal(t1.z, t2.z)
    assert t1.grid_ctas > 1


def test_staged_and_unstaged_tiles_agree_bitwise(monkeypatch):
    from paper_2001_04179_b200.workloads import c1_matrix

    g = load("c1_golden.npz")
    prob = P.ProblemInstance(a=P.Matrix.from_dense(c1_matrix()), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=17, max_iters=200,
                         row_partition=P.contiguous_partition(2000, 100, "row"),
                         col_partition=P.contiguous_partition(500, 100, "col"),
                         stop=P.StoppingRule(mode="max_iters_only"), beta_max=float(g["beta"]))
    t1 = P.run(prob, cfg)
    monkeypatch.setenv("REBK_NO_STAGE", "1")
    t2 = P.run(prob, cfg)
    assert np.array_equal(t1.x, t2.x) and np.array_equal(t1.z, t2.z)


def c1_instance():
    from paper_2001_04179_b200.workloads import c1_matrix

    g = load("c1_golden.npz")
    a = c1_matrix()
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(2000, 100, "row"), P.contiguous_partition(500, 100, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=int(g["seed"]), max_iters=50_000,
                         row_partition=rp, col_partition=cp, stop=P.StoppingRule(tol=float(g["tol"])),
                         beta_max=float(g["beta"]))
    return g, a, prob, cfg


def test_c1_full_run_matches_reference():
    g, a, prob, cfg = c1_instance()
    tr = P.run(prob, cfg)
    k = int(g["iters"])
    assert tr.converged and tr.iters == k == 547
    assert rel(tr.x, g[f"x_{k}"]) <= RTOL
    assert rel(tr.z, g[f"z_{k}"]) <= RTOL
    assert tr.final_error == pytest.approx(float(g["final_error"]), rel=1e-9)
    # in-process oracle on the same instance
    orc = OracleSolver(a, g["b"], np.arange(0, 2001, 100), np.arange(0, 501, 100), float(g["alpha"]))
    res = orc.run(int(g["seed"]), 50_000, float(g["tol"]), g["x_star"])
    assert res["iters"] == tr.iters
    assert rel(tr.x, res["x"]) <= RTOL and rel(tr.z, res["z"]) <= RTOL


def test_c1_step_snapshots():
    g, a, prob, cfg = c1_instance()
    ctx = P.prepare(prob, cfg)
    st = ctx.initial_state()
    for k in range(1, 101):
        ctx.step(st)
        if k in (1, 10, 100):
            assert rel(st.x, g[f"x_{k}"]) <= RTOL
            assert rel(st.z, g[f"z_{k}"]) <= RTOL


def test_device_block_norms_match_host():
    _, a, prob, cfg = c1_instance()
    dm = prob.a.device()
    for axis, ptr, sl in ((0, np.arange(0, 2001, 100), lambda lo, hi: a[lo:hi]),
                          (1, np.arange(0, 501, 100), lambda lo, hi: a[:, lo:hi])):
        got = dm.block_frobenius_sq(axis, ptr)
        want = np.array([np.sum(sl(lo, hi) ** 2) for lo, hi in zip(ptr[:-1], ptr[1:])])
        np.testing.assert_allclose(got, want, rtol=1e-13)


@pytest.mark.slow
def test_c2_full_run_matches_reference():
    """BASELINE config 2 (the bench workload): 4000 x 10000, rank 2000,
    blocks 200/200, alpha = 1/beta_max, to ||x - x*|| <= 1e-6 ||x*||."""
    from paper_2001_04179_b200.workloads import c2_arrays

    g = load("c2_golden.npz")
    a, b, xs = c2_arrays()
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=xs, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(4000, 200, "row"), P.contiguous_partition(10000, 200, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=int(g["seed"]), max_iters=50_000,
                         row_partition=rp, col_partition=cp, stop=P.StoppingRule(tol=float(g["tol"])),
                         beta_max=float(g["beta"]))
    ctx = P.prepare(prob, cfg)
    want = g["picks"].astype(np.int32)
    c = ctx.make_cfg(stop_mode="max_iters_only", tol=1.0, stride=1, max_iters=len(want),
                     key=_lib.philox_key(int(g["seed"])))
    out = np.empty((len(want), 2), dtype=np.int32)
    _lib.check(_lib.load().rebk_sample_sequence(ctypes.byref(c), 1, len(want),
                                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "sample")
    assert np.array_equal(out, want)
    tr = P.run(prob, cfg)
    k = int(g["iters"])
    assert tr.converged and tr.iters == k
    assert rel(tr.x, g[f"x_{k}"]) <= RTOL
    assert rel(tr.z, g[f"z_{k}"]) <= RTOL


def test_fast_path_taken_and_agrees_with_general_kernel(monkeypatch):
    """C1 runs on the clustered fast kernel; the general kernel (REBK_NO_FAST)
    reduces in a different fixed order, so the two agree to rounding only."""
    g, a, prob, cfg = c1_instance()
    t_fast = P.run(prob, cfg)
    assert t_fast.kernel_path in (1, 2, 6)
    monkeypatch.setenv("REBK_NO_FAST", "1")
    t_gen = P.run(prob, cfg)
    assert t_gen.kernel_path == 0
    assert t_fast.iters == t_gen.iters
    assert rel(t_fast.x, t_gen.x) <= 1e-12 and rel(t_fast.z, t_gen.z) <= 1e-12


def test_sparse_cases_bitwise_equal_to_reference():
    """The sparse kernel sums in scipy's order with unfused multiply/add, so
    its iterates equal the reference's bit for bit (tolerance kept as a
    fallback assertion only in the message)."""
    for case in [c for c in CASES if c.startswith("case_sp_")]:
        g = load(case)
        prob, cfg = case_problem(g)
        ctx = P.prepare(prob, cfg)
        st = ctx.initial_state()
        ks = set(int(k) for k in g["ks"])
        for k in range(1, max(ks) + 1):
            ctx.step(st)
            if k in ks:
                assert np.array_equal(st.x, g[f"x_{k}"]), (case, k, rel(st.x, g[f"x_{k}"]))
                if st.z is not None:
                    assert np.array_equal(st.z, g[f"z_{k}"]), (case, k, rel(st.z, g[f"z_{k}"]))


@pytest.mark.parametrize("env", [{}, {"REBK_CSR_SPEC": "0"}, {"REBK_CSR_STAGE": "0"}, {"REBK_CSR_PF": "0"},
                                 {"REBK_GRID": "3"}, {"REBK_GRID": "40"},
                                 {"REBK_CSR_SPEC": "0", "REBK_CSR_STAGE": "0", "REBK_CSR_PF": "0"}])
def test_sparse_kernel_variants_bitwise_equal_to_scipy_order(monkeypatch, env):
    """The CSR kernel's shared-memory staging of u / r, its L2 prefetch and
    its warp specialisation (and the fallbacks taken when a CTA's rows of I or
    columns of J fill all its warps: small grids) change where and when
    values are read, never the order they are summed in: a 12000 x 3000 sparse
    run (ragged blocks, stride 3, stop inside the run) equals the scipy-order
    oracle bit for bit under every switch."""
    import scipy.sparse as sp

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rs = np.random.default_rng(11)
    m, n = 12000, 3000
    a = sp.random(m, n, density=4e-3, format="csr", random_state=rs, data_rvs=rs.standard_normal)
    xs = rs.standard_normal(n)
    b = a @ xs + 1e-3 * rs.standard_normal(m)
    from scipy.sparse.linalg import lsqr

    x_star = lsqr(a, b, atol=1e-14, btol=1e-14, iter_lim=4000)[0]
    prob = P.ProblemInstance(a=P.Matrix.from_sparse(a), b=b, x_star=x_star, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(m, 700, "row"), P.contiguous_partition(n, 260, "col")
    tol = 0.5 * float(np.linalg.norm(x_star))
    cfg = P.SolverConfig(algorithm="rebk", alpha=1.2, seed=5, max_iters=600, row_partition=rp, col_partition=cp,
                         stop=P.StoppingRule(tol=tol, check_stride=3), beta_max=1.0)
    t = P.run(prob, cfg)
    assert t.kernel_path == 3
    rp_ptr = np.array(list(range(0, m, 700)) + [m])
    cp_ptr = np.array(list(range(0, n, 260)) + [n])
    orc = OracleSolver(a, b, rp_ptr, cp_ptr, cfg.alpha, algorithm="rebk")
    res = orc.run(5, 600, tol, x_star, stride=3)
    assert res["iters"] == t.iters and res["converged"] == t.converged
    assert 3 <= t.iters < 600 or not t.converged
    assert np.array_equal(t.x, res["x"]), rel(t.x, res["x"])
    assert np.array_equal(t.z, res["z"]), rel(t.z, res["z"])


@pytest.mark.slow
def test_c4_sparse_full_run_matches_reference():
    """BASELINE config 4: CSR 200000 x 50000, 1e7 nnz, blocks 2000/1000."""
    if not os.path.exists(os.path.join(GOLD, "c4_golden.npz")):
        pytest.skip("c4 golden vectors not generated")
    from paper_2001_04179_b200.workloads import c4_matrix

    g = load("c4_golden.npz")
    s, _ = c4_matrix()
    prob = P.ProblemInstance(a=P.Matrix.from_sparse(s), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(200000, 2000, "row"), P.contiguous_partition(50000, 1000, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=int(g["seed"]), max_iters=50_000,
                         row_partition=rp, col_partition=cp, stop=P.StoppingRule(tol=float(g["tol"])),
                         beta_max=float(g["beta"]))
    tr = P.run(prob, cfg)
    k = int(g["iters"])
    assert tr.kernel_path == 3
    assert tr.converged and tr.iters == k
    assert rel(tr.x, g[f"x_{k}"]) <= RTOL
    assert rel(tr.z, g[f"z_{k}"]) <= RTOL


def test_multi_rhs_fp32_matches_reference_columns():
    """Config-5 family (fp32, 8 RHS sharing one block sequence): per-column
    ITER equal to the reference's fp64 single-RHS runs (±1 for fp32 rounding
    at the threshold) and X at the common final iteration within 1e-4."""
    from paper_2001_04179_b200.multirhs import run_multi
    from paper_2001_04179_b200.workloads import c5_arrays

    g = load("c5mini_golden.npz")
    a32, b32, xs = c5_arrays(6000, 600, 8)
    rp, cp = P.contiguous_partition(6000, 64, "row"), P.contiguous_partition(600, 64, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=17, max_iters=50_000, row_partition=rp,
                         col_partition=cp, stop=P.StoppingRule(tol=1.0), beta_max=float(g["beta"]))
    tr = run_multi(a32, b32, cfg, X_star=xs, tols=g["tols"])
    assert tr.converged
    assert np.all(np.abs(tr.iters_per_rhs - g["iters"]) <= 1), (tr.iters_per_rhs, g["iters"])
    assert abs(tr.iters - int(g["K"])) <= 1
    if tr.iters == int(g["K"]):
        for c in range(2):
            assert rel(tr.X[:, c], g["x_K"][:, c]) <= 1e-4


def test_multi_rhs_device_block_weights_give_the_reference_sequence():
    """run_multi's default sampler arrays: block weights from the device's
    fp32 copy of A (fp64 accumulation) against the reference's arithmetic on
    the host upcast (`flat @ flat` per block): equal to rounding, and the
    block sequences drawn from the two sets of arrays are identical; X and Z
    after 200 iterations agree to fp32 rounding on either route."""
    from paper_2001_04179_b200.multirhs import DeviceMatrix32, _DeviceWeightsContext, run_multi
    from paper_2001_04179_b200.solvers import SolverContext
    from paper_2001_04179_b200.workloads import c5_arrays

    g = load("c5mini_golden.npz")
    a32, b32, xs = c5_arrays(6000, 600, 8)
    # ragged last blocks on both axes
    rp, cp = P.contiguous_partition(6000, 70, "row"), P.contiguous_partition(600, 64, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=17, max_iters=200, row_partition=rp,
                         col_partition=cp, stop=P.StoppingRule(mode="max_iters_only"), beta_max=float(g["beta"]))
    a64 = P.Matrix.from_dense(a32.astype(np.float64))
    prob = P.ProblemInstance(a=a64, b=b32[:, 0].astype(np.float64), x_star=None, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    host = SolverContext(prob, cfg)
    dm = DeviceMatrix32(a32)
    dev = _DeviceWeightsContext(dm, 6000, 600, cfg)
    assert np.allclose(dev.row_sampler.weights, host.row_sampler.weights, rtol=1e-13, atol=0.0)
    assert np.allclose(dev.col_sampler.weights, host.col_sampler.weights, rtol=1e-13, atol=0.0)
    picks = []
    for ctx in (host, dev):
        c = ctx.make_cfg(stop_mode="max_iters_only", tol=1.0, stride=1, max_iters=20000, key=_lib.philox_key(17))
        out = np.empty(2 * 20000, dtype=np.int32)
        _lib.check(_lib.load().rebk_sample_sequence(ctypes.byref(c), 1, 20000,
                                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))),
                   "rebk_sample_sequence")
        picks.append(out)
    assert np.array_equal(picks[0], picks[1])
    t_dev = run_multi(a32, b32, cfg, device_matrix=dm)
    t_host = run_multi(a32, b32, cfg, device_matrix=dm, a64=a64)
    assert t_dev.iters == t_host.iters == 200
    assert rel(t_dev.X, t_host.X) <= 1e-6 and rel(t_dev.Z, t_host.Z) <= 1e-6


@pytest.mark.slow
def test_multi_rhs_fp32_baseline_c5_matches_reference_columns():
    """BASELINE config 5 at its stated size: fp32 A = randn(50000, 5000), 64
    right-hand sides, blocks of 256 (ragged last blocks of 80 rows and 136
    columns).  Against 64 fp64 kaczmarz.run() calls of the reference on the
    fp64 upcast (tests/golden/c5_golden.npz, gen_golden.py --c5-full):
    every column's ITER within +-1 (fp32 rounding at the threshold), the run's
    K = max ITER within +-1, and for columns 0, 1, 63 X after exactly the
    reference's K iterations within the north star's 1e-4."""
    from paper_2001_04179_b200.multirhs import DeviceMatrix32, run_multi
    from paper_2001_04179_b200.workloads import c5_arrays

    g = load("c5_golden.npz")
    cols = [int(c) for c in g["cols"]]
    a32, b32, xs = c5_arrays()
    assert a32.shape == (50000, 5000) and b32.shape == (50000, 64)
    # the pinned columns exactly as the reference ran them (the rest of B
    # only differs from the generator's by host LAPACK/BLAS rounding)
    b32 = np.array(b32)
    xs = np.array(xs)
    b32[:, cols] = g["b_cols"]
    xs[:, cols] = g["x_star_cols"]
    a64 = P.Matrix.from_dense(a32.astype(np.float64))
    rp, cp = P.contiguous_partition(50000, 256, "row"), P.contiguous_partition(5000, 256, "col")
    assert rp.block_sizes()[-1] == 80 and cp.block_sizes()[-1] == 136
    dm = DeviceMatrix32(a32)
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=17, max_iters=50_000, row_partition=rp,
                         col_partition=cp, stop=P.StoppingRule(tol=1.0), beta_max=float(g["beta"]))
    tr = run_multi(a32, b32, cfg, X_star=xs, tols=g["tols"], device_matrix=dm, a64=a64)
    assert tr.kernel_path == 8  # the hand-written tcgen05 kernel, not a library fallback
    assert tr.converged
    d = np.abs(tr.iters_per_rhs - g["iters"])
    assert np.all(d <= 1), (np.flatnonzero(d > 1), tr.iters_per_rhs[d > 1], g["iters"][d > 1])
    K = int(g["K"])
    assert abs(tr.iters - K) <= 1
    cfgK = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=17, max_iters=K, row_partition=rp,
                          col_partition=cp, stop=P.StoppingRule(mode="max_iters_only"), beta_max=float(g["beta"]))
    tK = run_multi(a32, b32, cfgK, device_matrix=dm, a64=a64)
    assert tK.iters == K
    for j, c in enumerate(cols):
        assert rel(tK.X[:, c], g["x_K"][:, j]) <= 1e-4, (c, rel(tK.X[:, c], g["x_K"][:, j]))


def _mini_mrhs(algorithm="rebk", blk=64, m=6000, n=600, R=8, max_iters=40, stride=1, mode="max_iters_only"):
    from paper_2001_04179_b200.multirhs import DeviceMatrix32
    from paper_2001_04179_b200.workloads import c5_arrays

    a32, b32, xs = c5_arrays(m, n, R)
    rp = P.contiguous_partition(m, blk, "row")
    cp = P.contiguous_partition(n, blk, "col") if algorithm in ("rebk", "rek") else None
    a64 = P.Matrix.from_dense(a32.astype(np.float64))
    beta = 0.02
    kw = dict(algorithm=algorithm, alpha=1.0 / beta, seed=17, max_iters=max_iters, row_partition=rp,
              stop=P.StoppingRule(mode=mode, tol=1.0, check_stride=stride), beta_max=beta)
    if cp is not None:
        kw["col_partition"] = cp
    return a32, b32, xs, a64, DeviceMatrix32(a32), P.SolverConfig(**kw)


@pytest.mark.parametrize("algorithm,blk", [("rebk", 64), ("rebk", 100), ("rebk", 256), ("rabk", 64)])
def test_multi_rhs_persistent_kernel_matches_per_product_kernels(monkeypatch, algorithm, blk):
    """The persistent whole-run tcgen05 kernel (default) and the per-product
    kernels compute the same iteration: X (and Z) after 40 iterations agree
    to fp32 rounding of the different split-K orders; the persistent kernel
    replays bit for bit.  Ragged blocks (100), blocks wider than one 128-row
    MMA tile (256) and the no-column-sweep RABK variant included."""
    from paper_2001_04179_b200.multirhs import run_multi

    a32, b32, xs, a64, dm, cfg = _mini_mrhs(algorithm, blk)
    monkeypatch.setenv("REBK_MRHS_PK", "1")
    t1 = run_multi(a32, b32, cfg, device_matrix=dm, a64=a64)
    t1b = run_multi(a32, b32, cfg, device_matrix=dm, a64=a64)
    monkeypatch.setenv("REBK_MRHS_PK", "0")
    t0 = run_multi(a32, b32, cfg, device_matrix=dm, a64=a64)
    assert t1.iters == t0.iters == 40
    assert np.array_equal(t1.X, t1b.X)
    assert rel(t1.X, t0.X) <= 1e-5
    if algorithm == "rebk":
        assert np.array_equal(t1.Z, t1b.Z)
        assert rel(t1.Z, t0.Z) <= 1e-5


def test_multi_rhs_persistent_stop_state(monkeypatch):
    """Per-column stopping inside the persistent kernel: with a check stride
    of 7 the run ends at the first multiple of 7 (or max_iters) at which
    every column has crossed, and X at that iteration equals a
    max_iters-only run of exactly that many iterations."""
    from paper_2001_04179_b200.multirhs import run_multi

    g = load("c5mini_golden.npz")
    a32, b32, xs, a64, dm, cfg = _mini_mrhs("rebk", 64, max_iters=50_000, stride=7, mode="oracle_error")
    cfg.alpha = float(g["alpha"])
    monkeypatch.setenv("REBK_MRHS_PK", "1")
    t = run_multi(a32, b32, cfg, X_star=xs, tols=g["tols"], device_matrix=dm, a64=a64)
    assert t.converged and t.iters % 7 == 0
    assert np.all(t.iters_per_rhs % 7 == 0) and t.iters == t.iters_per_rhs.max()
    assert np.all(np.abs(t.iters_per_rhs - g["iters"]) <= 7)
    cfg2 = P.SolverConfig(algorithm="rebk", alpha=cfg.alpha, seed=17, max_iters=int(t.iters),
                          row_partition=cfg.row_partition, col_partition=cfg.col_partition,
                          stop=P.StoppingRule(mode="max_iters_only"), beta_max=cfg.beta_max)
    t2 = run_multi(a32, b32, cfg2, device_matrix=dm, a64=a64)
    assert np.array_equal(t.X, t2.X) and np.array_equal(t.Z, t2.Z)


@pytest.mark.parametrize("ranks", [1, 2, 4])
def test_sharded_kernels_c1(ranks):
    """Config-3 layout (interleaved row shards, u and dx allreduced) on the
    C1 instance: one real rank, or 2/4 virtual ranks in lockstep on one GPU.
    Same ITER as the reference and iterates within 1e-10."""
    from paper_2001_04179_b200.sharded import CudaShardBackend, owned_rows, plan_from_context, run_virtual_ranks

    g, a, prob, cfg = c1_instance()
    ctx = P.prepare(prob, cfg)
    plan = plan_from_context(ctx, 2000)
    owns = [owned_rows(ctx._row_ptr, ranks, r) for r in range(ranks)]
    bes = [CudaShardBackend(a[rows], prob.b[rows], g["x_star"], True) for rows, _ in owns]
    res = run_virtual_ranks(bes, plan, [rg for _, rg in owns], 2000, float(g["tol"]))
    k = int(g["iters"])
    assert res["converged"] and res["iters"] == k
    z = np.zeros(2000)
    for (rows, _), (x, zl) in zip(owns, res["states"]):
        assert rel(x, g[f"x_{k}"]) <= RTOL
        z[rows] = zl
    assert rel(z, g[f"z_{k}"]) <= RTOL


@pytest.mark.parametrize("split", ["1", "0"])
def test_split_and_fused_paths_match_reference_c1(monkeypatch, split):
    """The split (column group -> row group) kernel and the fused fast kernel
    both reproduce the reference's C1 run: ITER, x and z within 1e-10, and
    bitwise replay."""
    monkeypatch.setenv("REBK_SPLIT", split)
    g, a, prob, cfg = c1_instance()
    t1 = P.run(prob, cfg)
    t2 = P.run(prob, cfg)
    assert t1.kernel_path == (6 if split == "1" else 2) or t1.kernel_path in (1, 2, 6)
    k = int(g["iters"])
    assert t1.converged and t1.iters == k
    assert rel(t1.x, g[f"x_{k}"]) <= RTOL and rel(t1.z, g[f"z_{k}"]) <= RTOL
    assert np.array_equal(t1.x, t2.x) and np.array_equal(t1.z, t2.z)


def test_split_path_small_ring_and_chunk_edges(monkeypatch):
    """Ring depth 2 (column group throttled hard) and a max_iters that is
    not converged: the stop state must still be the exact iteration."""
    monkeypatch.setenv("REBK_SPLIT_RING", "2")
    g, a, prob, cfg = c1_instance()
    t = P.run(prob, cfg)
    k = int(g["iters"])
    assert t.iters == k and rel(t.x, g[f"x_{k}"]) <= RTOL and rel(t.z, g[f"z_{k}"]) <= RTOL
    cfg2 = P.SolverConfig(algorithm="rebk", alpha=cfg.alpha, seed=cfg.seed, max_iters=100,
                          row_partition=cfg.row_partition, col_partition=cfg.col_partition,
                          stop=P.StoppingRule(mode="max_iters_only"), beta_max=cfg.beta_max)
    t2 = P.run(prob, cfg2)
    assert t2.iters == 100 and rel(t2.x, g["x_100"]) <= RTOL and rel(t2.z, g["z_100"]) <= RTOL


@pytest.mark.parametrize("grid", ["0", "7"])
def test_stream_path_matches_reference_c1(monkeypatch, grid):
    """The streaming kernel (TMA ring, used when block slices exceed shared
    memory, e.g. C3) forced onto C1: ITER, x, z as the reference, bitwise
    replay; with 7 CTAs each column slice is ~286 rows = 13 ring boxes."""
    monkeypatch.setenv("REBK_NO_FAST", "1")
    monkeypatch.setenv("REBK_STREAM", "2")
    if grid != "0":
        monkeypatch.setenv("REBK_GRID", grid)
    g, a, prob, cfg = c1_instance()
    t1 = P.run(prob, cfg)
    t2 = P.run(prob, cfg)
    assert t1.kernel_path == 7
    k = int(g["iters"])
    assert t1.converged and t1.iters == k
    assert rel(t1.x, g[f"x_{k}"]) <= RTOL and rel(t1.z, g[f"z_{k}"]) <= RTOL
    assert np.array_equal(t1.x, t2.x) and np.array_equal(t1.z, t2.z)


@pytest.mark.parametrize("env", [{"REBK_STREAM_ORDER": "1"}, {"REBK_STREAM_ORDER": "1", "REBK_STREAM_TAIL": "2"},
                                 {"REBK_STREAM_TAIL": "3"}, {"REBK_STREAM_DBG": "1"}])
def test_stream_path_schedule_variants_bitwise(monkeypatch, env):
    """The streaming kernel's pass order within a step, its L2 retention of
    C1's tail and an extra barrier per step move boxes and barriers around,
    not arithmetic: ITER, x and z equal the default
    schedule's bit for bit (and the reference's within 1e-10).  (A different
    ring depth or walk direction changes the summation order.)"""
    monkeypatch.setenv("REBK_NO_FAST", "1")
    monkeypatch.setenv("REBK_STREAM", "2")
    g, a, prob, cfg = c1_instance()
    t0 = P.run(prob, cfg)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    t1 = P.run(prob, cfg)
    assert t0.kernel_path == 7 and t1.kernel_path == 7
    k = int(g["iters"])
    assert t1.converged and t1.iters == k == t0.iters
    assert np.array_equal(t0.x, t1.x) and np.array_equal(t0.z, t1.z)
    assert rel(t1.x, g[f"x_{k}"]) <= RTOL and rel(t1.z, g[f"z_{k}"]) <= RTOL


@pytest.mark.parametrize("algorithm", ["rebk", "rabk", "rk", "rek"])
def test_stream_path_ragged_blocks_and_algorithms(monkeypatch, algorithm):
    """Ragged partitions (odd block widths, a short last block), an odd n,
    stride 3 and max_iters cut-off on the streaming kernel vs the oracle."""
    monkeypatch.setenv("REBK_NO_FAST", "1")
    monkeypatch.setenv("REBK_STREAM", "2")
    rs = np.random.default_rng(5)
    m, n = 701, 333
    a = rs.standard_normal((m, n))
    xs = rs.standard_normal(n)
    b = a @ xs + 0.01 * rs.standard_normal(m)
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=np.linalg.lstsq(a, b, rcond=None)[0],
                             b_perp=None, meta=P.ProblemMeta(0, None, False, 0, 0.0))
    single = algorithm in ("rek", "rk")
    rp = P.contiguous_partition(m, 1 if single else 97, "row")
    cp = P.contiguous_partition(n, 1 if single else 61, "col")
    cfg = P.SolverConfig(algorithm=algorithm, alpha=1.0 if single else 0.7, seed=3, max_iters=400,
                         row_partition=rp, col_partition=cp, stop=P.StoppingRule(tol=1e-9, check_stride=3),
                         beta_max=1.0)
    t = P.run(prob, cfg)
    assert t.kernel_path == 7
    rp_ptr = np.arange(m + 1) if single else np.array(list(range(0, m, 97)) + [m])
    cp_ptr = np.arange(n + 1) if single else np.array(list(range(0, n, 61)) + [n])
    orc = OracleSolver(a, b, rp_ptr, cp_ptr, cfg.alpha, algorithm=algorithm)
    res = orc.run(3, 400, 1e-9, prob.x_star, stride=3)
    assert res["iters"] == t.iters and res["converged"] == t.converged
    assert rel(t.x, res["x"]) <= 1e-10
    if algorithm in ("rebk", "rek"):
        assert rel(t.z, res["z"]) <= 1e-10


def test_odd_column_block_starts_take_a_safe_path():
    """Column blocks of 99 (odd starts): the clustered kernels need 16-byte
    aligned TMA starts and must not be chosen; the result still matches the
    oracle."""
    g, a, prob, _ = c1_instance()
    rp, cp = P.contiguous_partition(2000, 100, "row"), P.contiguous_partition(500, 99, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=int(g["seed"]), max_iters=300,
                         row_partition=rp, col_partition=cp, stop=P.StoppingRule(mode="max_iters_only"),
                         beta_max=float(g["beta"]))
    t = P.run(prob, cfg)
    assert t.kernel_path in (0, 7)
    orc = OracleSolver(a, g["b"], np.arange(0, 2001, 100), np.array(list(range(0, 500, 99)) + [500]),
                       float(g["alpha"]))
    res = orc.run(int(g["seed"]), 300, 0.0, None, mode="max_iters_only")
    assert rel(t.x, res["x"]) <= RTOL and rel(t.z, res["z"]) <= RTOL


@pytest.mark.slow
def test_c3_full_size_matches_oracle():
    """BASELINE config 3 at full size (200000 x 10000, 16 GB, built on the
    device): the streaming kernel's run to ||x - x*|| <= 1e-6 ||x*|| against
    the oracle on the same instance: ITER equal, x and z within 1e-10."""
    import torch

    from oracle.rebk_oracle import NumpyRng
    from paper_2001_04179_b200.matrix import DeviceMatrix
    from paper_2001_04179_b200.workloads import c3_device

    wl = c3_device()
    m, n = wl.shape
    dm = DeviceMatrix.from_device_pointer(wl.a.data_ptr(), m, n, n, 0)
    tol = wl.rel_tol * float(wl.x_star.norm())
    c = wl.cfg("oracle_error", tol, 2000)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    z = wl.b.clone()
    tr = _lib.RebkTrace()
    _lib.check(_lib.load().rebk_run_device(dm.handle, ctypes.byref(c), ctypes.c_void_p(wl.b.data_ptr()),
                                           ctypes.c_void_p(wl.x_star.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                           ctypes.c_void_p(z.data_ptr()), None, ctypes.byref(tr)), "run")
    assert tr.kernel_path == 7 and tr.converged
    a_h = wl.a.cpu().numpy()
    orc = OracleSolver(a_h, wl.b.cpu().numpy(), wl.row_ptr, wl.col_ptr, wl.alpha, "rebk")
    res = orc.run(wl.seed, 2000, tol, wl.x_star.cpu().numpy(), rng=NumpyRng(wl.seed))
    assert res["iters"] == tr.iters
    assert rel(x.cpu().numpy(), res["x"]) <= RTOL and rel(z.cpu().numpy(), res["z"]) <= RTOL


def test_sharded_chunked_loop_over_nccl_c1():
    """The multi-GPU driver as bench.py runs it (one process per GPU, NCCL
    allreduces through torch.distributed, errors checked on the device once
    per chunk with replay to the exact crossing) at world size 1 on the C1
    instance: same ITER as the reference and iterates within 1e-10."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2001_04179_b200.sharded import (CudaShardBackend, owned_rows, plan_from_context,
                                                run_sharded_chunked)

    g, a, prob, cfg = c1_instance()
    ctx = P.prepare(prob, cfg)
    plan = plan_from_context(ctx, 2000)
    rows, ranges = owned_rows(ctx._row_ptr, 1, 0)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        dev = torch.device("cuda", 0)
        t = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
        be = CudaShardBackend.from_device(t(a[rows]), t(prob.b[rows]), t(g["x_star"]), True, 0)
        res = run_sharded_chunked(be, plan, ranges, 2000, float(g["tol"]), allreduce=lambda v: dist.all_reduce(v),
                                  chunk=32)
    finally:
        dist.destroy_process_group()
    k = int(g["iters"])
    assert res["converged"] and res["iters"] == k
    assert rel(res["x"], g[f"x_{k}"]) <= RTOL
    z = np.zeros(2000)
    z[rows] = res["z_local"]
    assert rel(z, g[f"z_{k}"]) <= RTOL


def test_sharded_native_nccl_runner_c1():
    """rebk_shard_run (the whole sharded loop in C++, NCCL loaded by librebk,
    world size 1) on the C1 instance: same ITER as the reference and iterates
    within 1e-10."""
    import torch

    from paper_2001_04179_b200.sharded import (CudaShardBackend, NcclComm, nccl_unique_id, owned_rows,
                                                plan_from_context, run_sharded_native)

    g, a, prob, cfg = c1_instance()
    ctx = P.prepare(prob, cfg)
    plan = plan_from_context(ctx, 2000)
    rows, ranges = owned_rows(ctx._row_ptr, 1, 0)
    dev = torch.device("cuda", 0)
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    comm = NcclComm(nccl_unique_id(), 1, 0, 0)
    try:
        for chunk in (32, 7):
            be = CudaShardBackend.from_device(t(a[rows]), t(prob.b[rows]), t(g["x_star"]), True, 0)
            res = run_sharded_native(be, comm, plan, ranges, 2000, float(g["tol"]), chunk=chunk)
            k = int(g["iters"])
            assert res["converged"] and res["iters"] == k, (chunk, res["iters"])
            assert rel(res["x"], g[f"x_{k}"]) <= RTOL
            z = np.zeros(2000)
            z[rows] = res["z_local"]
            assert rel(z, g[f"z_{k}"]) <= RTOL
    finally:
        comm.close()


@pytest.mark.parametrize("algorithm", ["rebk", "rabk"])
def test_sharded_native_equals_python_loop(algorithm):
    """The C++ issue loop (rebk_shard_run) and the Python loop
    (run_sharded_chunked over torch.distributed) launch the same kernels in
    the same order: identical ITER and bitwise-identical iterates, for REBK
    and for RABK (no column sweep), with a check stride and a chunk that
    does not divide it."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2001_04179_b200.sharded import (CudaShardBackend, NcclComm, nccl_unique_id, owned_rows,
                                                plan_from_context, run_sharded_chunked, run_sharded_native)

    g, a, prob, cfg = c1_instance()
    cfg.algorithm = algorithm
    if algorithm == "rabk":
        cfg.col_partition = None
    ctx = P.prepare(prob, cfg)
    plan = plan_from_context(ctx, 3000)
    rows, ranges = owned_rows(ctx._row_ptr, 1, 0)
    dev = torch.device("cuda", 0)
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    ext = algorithm == "rebk"
    tol, stride = float(g["tol"]), 3
    comm = NcclComm(nccl_unique_id(), 1, 0, 0)
    try:
        be = CudaShardBackend.from_device(t(a[rows]), t(prob.b[rows]), t(g["x_star"]), ext, 0)
        nat = run_sharded_native(be, comm, plan, ranges, 3000, tol, stride=stride, chunk=10)
    finally:
        comm.close()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        be = CudaShardBackend.from_device(t(a[rows]), t(prob.b[rows]), t(g["x_star"]), ext, 0)
        py = run_sharded_chunked(be, plan, ranges, 3000, tol, stride=stride, allreduce=lambda v: dist.all_reduce(v),
                                 chunk=10)
    finally:
        dist.destroy_process_group()
    assert nat["converged"] == py["converged"] and nat["iters"] == py["iters"]
    assert nat["iters"] % stride == 0
    assert np.array_equal(nat["x"], py["x"])
    if ext:
        assert np.array_equal(nat["z_local"], py["z_local"])


@pytest.mark.parametrize("max_iters,stride", [(0, 1), (200, 10), (205, 10), (37, 1)])
def test_run_budget_and_checkpoint_semantics_c1(max_iters, stride):
    """run() semantics of solvers.py:425-474 on the device path (split kernel,
    C1): a zero budget stops after the k = 0 check; checks every `stride`
    iterations plus a final one when max_iters is not a multiple of it;
    recorded errors and checkpoints, x and z equal the CPU restatement's."""
    g, a, prob, cfg = c1_instance()
    cfg.max_iters = max_iters
    cfg.stop = P.StoppingRule(tol=1e-300, check_stride=stride)
    cfg.record_errors = True
    tr = P.run(prob, cfg)
    orc = OracleSolver(a, prob.b, cfg.row_partition.pointers(), cfg.col_partition.pointers(), cfg.alpha, "rebk")
    res = orc.run(int(g["seed"]), max_iters, 1e-300, g["x_star"], stride=stride, record=True)
    assert not tr.converged and tr.iters == res["iters"] == max_iters
    want = list(range(0, max_iters + 1, stride))
    if max_iters % stride:
        want.append(max_iters)
    assert tr.checkpoints.tolist() == res["checkpoints"].tolist() == want
    np.testing.assert_allclose(tr.errors, res["errors"], rtol=1e-10, atol=0)
    assert tr.final_error == pytest.approx(float(res["errors"][-1]), rel=1e-10)
    if max_iters == 0:
        assert np.all(tr.x == 0.0) and np.array_equal(tr.z, prob.b)
    else:
        assert rel(tr.x, res["x"]) <= RTOL and rel(tr.z, res["z"]) <= RTOL


@pytest.mark.parametrize("with_z0", [False, True])
def test_warm_start_x0_z0_c1(with_z0):
    """Non-default starting points (SolverConfig.x0 / z0, solvers.py:231-265)
    through the device path: same iterates as the CPU restatement started
    from the same x0 (and z0)."""
    g, a, prob, cfg = c1_instance()
    rng = np.random.default_rng(5)
    x0 = 0.1 * rng.standard_normal(500)
    z0 = prob.b + 0.01 * rng.standard_normal(2000) if with_z0 else None
    cfg.x0, cfg.z0 = x0, z0
    cfg.max_iters = 150
    cfg.stop = P.StoppingRule(tol=1e-300, check_stride=5)
    tr = P.run(prob, cfg)
    orc = OracleSolver(a, prob.b, cfg.row_partition.pointers(), cfg.col_partition.pointers(), cfg.alpha, "rebk")
    res = orc.run(int(g["seed"]), 150, 1e-300, g["x_star"], stride=5, x0=x0, z0=z0)
    assert tr.iters == res["iters"] == 150
    assert rel(tr.x, res["x"]) <= RTOL and rel(tr.z, res["z"]) <= RTOL
    assert tr.final_error == pytest.approx(float(res["final_error"]), rel=1e-10)

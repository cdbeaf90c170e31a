"""Robustness of the device path: concurrent runs on one context (SPEC.md:390
"distinct runs on the same ProblemInstance may execute concurrently";
SPEC.md:84 matrices shared read-only between threads), NaN/Inf in the
stopping reduction (the reference keeps iterating; rebk_cfg.nonfinite_stop
makes the C-ABI stop with REBK_ENONFINITE), and the explicit report of the
multi-RHS library path."""

import ctypes
import os
import threading
import warnings

import numpy as np
import pytest

import paper_2001_04179_b200 as P
from paper_2001_04179_b200 import _lib

pytestmark = pytest.mark.gpu


def dense_problem(m=600, n=200, seed=1):
    g = np.random.default_rng(seed)
    a = g.standard_normal((m, n))
    xs = g.standard_normal(n)
    b = a @ xs + 0.05 * g.standard_normal(m)
    x_star = np.linalg.lstsq(a, b, rcond=None)[0]
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=x_star, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    return a, b, x_star, prob


def run_threads(fns):
    out = [None] * len(fns)
    errs = []

    def body(i):
        try:
            out[i] = fns[i]()
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)

    ts = [threading.Thread(target=body, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return out


@pytest.mark.parametrize("seed_pair", [(5, 5), (5, 6)])
def test_concurrent_dense_runs_on_one_matrix(seed_pair):
    """Two host threads run solves on ONE Matrix (one shared device ctx,
    uploaded once under the matrix's lock) at the same time, each on its own
    stream; every result equals the same solve run alone, bit for bit."""
    a, b, xs, prob = dense_problem()
    rp, cp = P.contiguous_partition(600, 40, "row"), P.contiguous_partition(200, 40, "col")
    tol = 1e-9 * float(np.linalg.norm(xs))

    def cfg(seed):
        return P.SolverConfig(algorithm="rebk", alpha=1.0, seed=seed, max_iters=20000, row_partition=rp,
                              col_partition=cp, stop=P.StoppingRule(tol=tol), beta_max=0.3)

    alone = [P.run(prob, cfg(s)) for s in seed_pair]
    prob.a.release_device()
    both = run_threads([lambda s=s: P.run(prob, cfg(s)) for s in seed_pair] * 2)
    assert len(prob.a._device_cache) == 1  # one upload for all four runs
    for i, tr in enumerate(both):
        ref = alone[i % 2]
        assert tr.iters == ref.iters and np.array_equal(tr.x, ref.x) and np.array_equal(tr.z, ref.z)


def test_concurrent_sparse_runs_build_segment_lists_once():
    """Sparse: the first runs build the per-partition segment lists under
    the ctx mutex while another run wants the same lists."""
    import scipy.sparse as sp

    g = np.random.default_rng(2)
    s = sp.random(3000, 800, density=0.01, format="csr", random_state=g)
    s.data = g.standard_normal(s.nnz)
    xs = g.standard_normal(800)
    b = s @ xs + 0.01 * g.standard_normal(3000)
    prob = P.ProblemInstance(a=P.Matrix.from_sparse(s), b=b, x_star=xs, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(3000, 100, "row"), P.contiguous_partition(800, 50, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=1.0, seed=3, max_iters=300, row_partition=rp, col_partition=cp,
                         stop=P.StoppingRule(mode="max_iters_only"), beta_max=0.3)
    prob.a.device()  # ctx exists, no segment lists yet
    res = run_threads([lambda: P.run(prob, cfg) for _ in range(4)])
    for tr in res[1:]:
        assert np.array_equal(tr.x, res[0].x) and np.array_equal(tr.z, res[0].z)


def test_concurrent_multi_rhs_runs_share_transposed_copy():
    """fp32 ctx: the transposed copy of A is built once, under the mutex,
    and published only after it is complete; concurrent first runs agree."""
    from paper_2001_04179_b200.multirhs import DeviceMatrix32, run_multi
    from paper_2001_04179_b200.workloads import c5_arrays

    a32, b32, xs = c5_arrays(4000, 400, 8)
    a64 = P.Matrix.from_dense(a32.astype(np.float64))
    rp, cp = P.contiguous_partition(4000, 64, "row"), P.contiguous_partition(400, 64, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=20.0, seed=17, max_iters=60, row_partition=rp, col_partition=cp,
                         stop=P.StoppingRule(mode="max_iters_only"), beta_max=0.02)
    dm = DeviceMatrix32(a32)  # fresh: no transposed copy yet
    res = run_threads([lambda: run_multi(a32, b32, cfg, device_matrix=dm, a64=a64) for _ in range(3)])
    assert all(r.kernel_path == 8 for r in res)
    for r in res[1:]:
        assert np.array_equal(r.X, res[0].X)


def nonfinite_problem():
    a, b, xs, prob = dense_problem(seed=4)
    b = b.copy()
    b[7] = np.inf  # the reference validates A, not b (matrix.py:40-41)
    prob = P.ProblemInstance(a=prob.a, b=b, x_star=xs, b_perp=None, meta=prob.meta)
    rp, cp = P.contiguous_partition(600, 40, "row"), P.contiguous_partition(200, 40, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=1.0, seed=5, max_iters=50, row_partition=rp, col_partition=cp,
                         stop=P.StoppingRule(tol=1e-8), beta_max=0.3)
    return prob, cfg


def test_nonfinite_error_keeps_reference_semantics():
    """Like the reference's run(): no early stop, iters = max_iters, not
    converged, final error NaN; the trace says where it first appeared."""
    prob, cfg = nonfinite_problem()
    tr = P.run(prob, cfg)
    assert tr.iters == 50 and not tr.converged
    assert not np.isfinite(tr.final_error)
    assert tr.nonfinite_at == 1  # x0 = 0 is finite at the check of k = 0


def test_nonfinite_stop_returns_enonfinite_through_c_abi():
    prob, cfg = nonfinite_problem()
    ctx = P.prepare(prob, cfg)
    c = ctx.make_cfg(stop_mode="oracle_error", tol=1e-8, stride=1, max_iters=50, key=_lib.philox_key(5))
    c.nonfinite_stop = 1
    dm = prob.a.device()
    x = np.empty(200)
    z = np.empty(600)
    tr = _lib.RebkTrace()
    lib = _lib.load()
    rc = lib.rebk_run(dm.handle, ctypes.byref(c), _lib.dptr(prob.b), None, None, _lib.dptr(np.asarray(prob.x_star)),
                      _lib.dptr(x), _lib.dptr(z), ctypes.byref(tr))
    assert rc == -5 and b"non-finite" in lib.rebk_last_error()
    assert tr.iters == 1 and tr.nonfinite_at == 1 and not tr.converged
    with pytest.raises(_lib.NonFiniteError):
        _lib.check(rc, "rebk_run")


def test_multi_rhs_library_path_is_reported():
    """A shape outside the tcgen05 kernel's range (n not divisible by 4) runs
    the cuBLAS path, reported by kernel_path and a RuntimeWarning."""
    from paper_2001_04179_b200.multirhs import run_multi
    from paper_2001_04179_b200.workloads import c5_arrays

    a32, b32, xs = c5_arrays(1000, 202, 4)
    rp, cp = P.contiguous_partition(1000, 50, "row"), P.contiguous_partition(202, 50, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=10.0, seed=17, max_iters=20, row_partition=rp, col_partition=cp,
                         stop=P.StoppingRule(mode="max_iters_only"), beta_max=0.05)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        tr = run_multi(a32, b32, cfg)
    assert tr.kernel_path in (4, 5)
    assert any("cuBLAS" in str(x.message) for x in w)


@pytest.mark.parametrize("path_env,expect_path", [({}, 6), ({"REBK_SPLIT": "0"}, 2),
                                                  ({"REBK_NO_FAST": "1", "REBK_STREAM": "2"}, 7),
                                                  ({"REBK_RES_MIN_STRIDE": "1000"}, 0)])
def test_residual_proxy_on_the_fast_kernels(monkeypatch, path_env, expect_path):
    """residual_proxy stopping (solvers.py:410-421) on the split / fused /
    streaming kernels: they iterate in chunks of check_stride and stand-alone
    residual-check kernels decide between the chunks; same ITER, checkpoints,
    errors and iterates as the oracle (and as the general kernel)."""
    from oracle.rebk_oracle import OracleSolver
    from paper_2001_04179_b200.workloads import c1_matrix

    for k, v in path_env.items():
        monkeypatch.setenv(k, v)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1_golden.npz"))
    a = c1_matrix()
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(2000, 100, "row"), P.contiguous_partition(500, 100, "col")
    tol, stride = 1e-6, 10  # first crossing at k = 390
    # z0 = b + A v (with the default z0 = b the proxy is exactly 0 at k = 0)
    z0 = g["b"] + a @ (0.1 * np.random.default_rng(1).standard_normal(500))
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=17, max_iters=3000, row_partition=rp,
                         col_partition=cp, stop=P.StoppingRule(mode="residual_proxy", tol=tol, check_stride=stride),
                         record_errors=True, beta_max=float(g["beta"]), z0=z0)
    tr = P.run(prob, cfg)
    assert tr.kernel_path == expect_path
    orc = OracleSolver(a, g["b"], rp.pointers(), cp.pointers(), float(g["alpha"]), "rebk")
    ref = orc.run(17, 3000, tol, None, stride, "residual_proxy", z0=z0, record=True)
    assert ref["iters"] == 390
    assert tr.iters == ref["iters"] and tr.converged == ref["converged"] and ref["converged"]
    np.testing.assert_array_equal(tr.checkpoints, ref["checkpoints"])
    np.testing.assert_allclose(tr.errors, ref["errors"], rtol=1e-9)
    rel = lambda u, v: np.linalg.norm(u - v) / np.linalg.norm(v)
    assert rel(tr.x, ref["x"]) <= 1e-10 and rel(tr.z, ref["z"]) <= 1e-10


def test_resume_continues_a_run_bitwise():
    """resume(): a run cut at a budget and continued from its RunTrace (x, z,
    k; Philox stream advanced past the consumed draws) ends at the same
    iteration with bitwise the same iterates as the uninterrupted run
    (resume = (x, z, k))."""
    import dataclasses
    import os

    from paper_2001_04179_b200.workloads import c1_matrix

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1_golden.npz"))
    a = c1_matrix()
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(2000, 100, "row"), P.contiguous_partition(500, 100, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=int(g["seed"]), max_iters=50_000,
                         row_partition=rp, col_partition=cp, stop=P.StoppingRule(tol=float(g["tol"])),
                         beta_max=float(g["beta"]), record_errors=True)
    whole = P.run(prob, cfg)
    assert whole.converged and whole.iters == int(g["iters"])
    first = P.run(prob, dataclasses.replace(cfg, max_iters=200))
    assert not first.converged and first.iters == 200
    second = P.resume(prob, cfg, first)
    assert second.converged and second.iters == whole.iters
    assert np.array_equal(second.x, whole.x) and np.array_equal(second.z, whole.z)
    # the error curve of the continued leg is the tail of the whole run's
    assert int(second.checkpoints[0]) == 200 and int(second.checkpoints[-1]) == whole.iters
    assert np.array_equal(second.errors, whole.errors[200:])
    # a second cut, through a budget-only leg
    leg = P.resume(prob, dataclasses.replace(cfg, max_iters=400, stop=P.StoppingRule(mode="max_iters_only")), first)
    assert leg.iters == 400 and not leg.converged
    third = P.resume(prob, cfg, leg)
    assert third.iters == whole.iters and np.array_equal(third.x, whole.x) and np.array_equal(third.z, whole.z)
    with pytest.raises(ValueError):
        P.resume(prob, dataclasses.replace(cfg, stop=P.StoppingRule(tol=float(g["tol"]), check_stride=7)), first)

"""Randomized parity sweep: small random problems through the public API on
the B200 against the CPU oracle (which is pinned to the reference's golden
vectors in tests/test_oracle_golden.py).  Each seed draws a shape (tall,
wide, square, tiny), a density (dense or sparse), block sizes (ragged last
blocks, singleton blocks, one block), contiguous or shuffled index
partitions, an algorithm (rebk, rek, rabk, rk, dsbgs), a stopping mode
(oracle error, residual proxy, max_iters_only) and a check stride.  Gates:
same ITER / converged flag, same pick sequence, iterates within 1e-10
(sparse rebk: bitwise), final error within 1e-9 relative."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2001_04179_b200 as P
from oracle.rebk_oracle import NumpyRng, OracleSolver

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def blocks(g, length, shuffle):
    tau = int(g.choice([1, 2, 3, 5, 7, 16, 33, length]))
    tau = min(tau, length)
    idx = g.permutation(length) if shuffle else np.arange(length)
    return [np.sort(idx[i:i + tau]) for i in range(0, length, tau)]


def draw(seed):
    g = np.random.default_rng(1000 + seed)
    m = int(g.choice([3, 17, 40, 96, 250]))
    n = int(g.choice([2, 9, 31, 64, 120]))
    sparse = bool(g.random() < 0.3) and m * n >= 200
    if sparse:
        a = sp.random(m, n, density=0.25, format="lil", random_state=g, data_rvs=g.standard_normal)
        for r in range(m):  # no empty rows / columns
            a[r, r % n] = a[r, r % n] + 1.0
        for c in range(n):
            a[c % m, c] = a[c % m, c] + 1.0
        a = sp.csr_matrix(a)
        dense = a.toarray()
    else:
        dense = g.standard_normal((m, n))
        a = dense
    xs = g.standard_normal(n)
    b = dense @ xs + 0.1 * g.standard_normal(m)
    x_star = np.linalg.lstsq(dense, b, rcond=None)[0]
    algo = str(g.choice(["rebk", "rebk", "rek", "rabk", "rk", "dsbgs"]))
    shuffle = bool(g.random() < 0.3)
    rb = blocks(g, m, shuffle) if algo not in ("rk", "rek") else [np.array([i]) for i in range(m)]
    cb = None
    if algo in ("rebk", "dsbgs"):
        cb = blocks(g, n, shuffle)
    elif algo == "rek":
        cb = [np.array([j]) for j in range(n)]
    mode = str(g.choice(["oracle_error", "oracle_error", "residual_proxy", "max_iters_only"]))
    stride = int(g.choice([1, 1, 3, 10]))
    alpha = float(g.uniform(0.3, 1.2)) if algo not in ("rek", "rk") else 1.0
    if algo in ("rebk", "rabk", "dsbgs"):
        # a stable stepsize: alpha / ||block||^2 scaled by the largest block's spectral ratio bound (<= 1)
        alpha = float(g.uniform(0.3, 1.0))
    seed_s = int(g.integers(0, 2**31))
    max_iters = int(g.choice([0, 1, 7, 300, 2000]))
    tol = {"oracle_error": 1e-6 * float(np.linalg.norm(x_star)), "residual_proxy": 1e-6,
           "max_iters_only": 1.0}[mode]
    return dict(a=a, dense=dense, b=b, x_star=x_star, algo=algo, rb=rb, cb=cb, mode=mode, stride=stride,
                alpha=alpha, seed=seed_s, max_iters=max_iters, tol=tol, sparse=sparse)


@pytest.mark.parametrize("seed", range(40))
def test_random_problem_matches_oracle(seed):
    c = draw(seed)
    m, n = c["dense"].shape
    mat = P.Matrix.from_sparse(c["a"]) if c["sparse"] else P.Matrix.from_dense(c["a"])
    prob = P.ProblemInstance(a=mat, b=c["b"], x_star=c["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp = P.Partition("row", m, tuple(c["rb"]))
    cp = None if c["cb"] is None else P.Partition("col", n, tuple(c["cb"]))
    cfg = P.SolverConfig(algorithm=c["algo"], alpha=c["alpha"], seed=c["seed"], max_iters=c["max_iters"],
                         row_partition=rp, col_partition=cp, record_errors=True, beta_max=1e-300,
                         stop=P.StoppingRule(mode=c["mode"], tol=c["tol"], check_stride=c["stride"]))
    tr = P.run(prob, cfg)
    orc = OracleSolver(c["a"], c["b"], c["rb"], c["cb"], c["alpha"], c["algo"])
    ref = orc.run(c["seed"], c["max_iters"], c["tol"], c["x_star"], c["stride"], c["mode"], rng=NumpyRng(c["seed"]),
                  record=True)
    assert tr.iters == ref["iters"] and tr.converged == ref["converged"], (tr.iters, ref["iters"])
    if c["mode"] != "max_iters_only":
        np.testing.assert_array_equal(tr.checkpoints, ref["checkpoints"])
        np.testing.assert_allclose(tr.errors, ref["errors"], rtol=1e-9, atol=1e-14)
    assert rel(tr.x, ref["x"]) <= 1e-10, rel(tr.x, ref["x"])
    if ref["z"] is not None:
        assert rel(tr.z, ref["z"]) <= 1e-10, rel(tr.z, ref["z"])


_MIDSIZE_PATHS = {}


def draw_midsize(seed):
    """Mid-size dense problems of the shapes the clustered kernels take (the
    bench kernels of C1/C2: split column/row groups, fused; TMA tiles need
    even column-block starts) and the streaming kernel: ragged last blocks,
    row blocks of any width, strides, budgets that end between checks."""
    g = np.random.default_rng(7000 + seed)
    m = int(g.choice([640, 1100, 2000, 3001]))
    n = int(g.choice([256, 500, 750, 1024]))
    a = g.standard_normal((m, n))
    xs = g.standard_normal(n)
    b = a @ xs + 0.1 * g.standard_normal(m)
    x_star = np.linalg.lstsq(a, b, rcond=None)[0]
    tau_r = int(g.choice([37, 64, 100, 128, 250]))
    tau_c = int(g.choice([50, 64, 100, 126]))  # even: every column block starts on an even column
    algo = str(g.choice(["rebk", "rebk", "rebk", "rabk"]))
    mode = str(g.choice(["oracle_error", "oracle_error", "max_iters_only", "residual_proxy"]))
    stride = int(g.choice([1, 1, 4, 16]))
    max_iters = int(g.choice([150, 333, 600]))
    tol = {"oracle_error": 1e-3 * float(np.linalg.norm(x_star)), "residual_proxy": 1e-3, "max_iters_only": 1.0}[mode]
    return dict(a=a, b=b, x_star=x_star, tau_r=tau_r, tau_c=tau_c, algo=algo, mode=mode, stride=stride,
                max_iters=max_iters, tol=tol, alpha=float(g.uniform(0.8, 1.6)), seed=int(g.integers(0, 2**31)))


@pytest.mark.parametrize("seed", range(16))
def test_random_midsize_problem_on_the_fast_kernels_matches_oracle(seed):
    c = draw_midsize(seed)
    m, n = c["a"].shape
    prob = P.ProblemInstance(a=P.Matrix.from_dense(c["a"]), b=c["b"], x_star=c["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp = P.contiguous_partition(m, c["tau_r"], "row")
    cp = P.contiguous_partition(n, c["tau_c"], "col") if c["algo"] == "rebk" else None
    cfg = P.SolverConfig(algorithm=c["algo"], alpha=c["alpha"], seed=c["seed"], max_iters=c["max_iters"],
                         row_partition=rp, col_partition=cp, record_errors=True, beta_max=1e-300,
                         stop=P.StoppingRule(mode=c["mode"], tol=c["tol"], check_stride=c["stride"]))
    tr = P.run(prob, cfg)
    rb = [np.arange(i, min(i + c["tau_r"], m)) for i in range(0, m, c["tau_r"])]
    cb = None if cp is None else [np.arange(j, min(j + c["tau_c"], n)) for j in range(0, n, c["tau_c"])]
    orc = OracleSolver(c["a"], c["b"], rb, cb, c["alpha"], c["algo"])
    ref = orc.run(c["seed"], c["max_iters"], c["tol"], c["x_star"], c["stride"], c["mode"], rng=NumpyRng(c["seed"]),
                  record=True)
    assert tr.iters == ref["iters"] and tr.converged == ref["converged"], (tr.iters, ref["iters"], tr.kernel_path)
    if c["mode"] != "max_iters_only":
        np.testing.assert_array_equal(tr.checkpoints, ref["checkpoints"])
        np.testing.assert_allclose(tr.errors, ref["errors"], rtol=1e-9, atol=1e-14)
    assert rel(tr.x, ref["x"]) <= 1e-10, (rel(tr.x, ref["x"]), tr.kernel_path)
    if ref["z"] is not None:
        assert rel(tr.z, ref["z"]) <= 1e-10, (rel(tr.z, ref["z"]), tr.kernel_path)
    _MIDSIZE_PATHS[seed] = (tr.kernel_path, tr.grid_ctas, m, n, c["algo"], c["mode"])


def test_midsize_sweep_exercises_the_fast_kernels():
    """The sweep above is there for the bench kernels: it must have reached
    the split kernel (path 6) and a fused / streaming one, not only the
    general kernel (which small grids and short residual strides select)."""
    if len(_MIDSIZE_PATHS) < 16:
        pytest.skip("runs after the whole mid-size sweep")
    paths = {v[0] for v in _MIDSIZE_PATHS.values()}
    assert 6 in paths, _MIDSIZE_PATHS
    assert paths & {1, 2, 7}, _MIDSIZE_PATHS

"""Pin the CPU oracle against the reference's own outputs (no GPU).

The golden vectors in tests/golden/ were produced by running the reference
package (tests/golden/gen_golden.py).  Here the oracle restatement must
reproduce them: the random stream and block-index sequence exactly, the
iterates to 1e-12 (bitwise on the generating machine; a different BLAS on
another host may reorder a dot product).
"""

import glob
import os

import numpy as np
import pytest

from oracle.rebk_oracle import OracleRng, OracleSolver, seedseq_state_u64

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=True)


def test_reference_pinned_stream_values():
    # test_sampling.py:161-166 pins these three draws of Rng(2024), abs=0.0
    r = OracleRng(2024)
    assert [r.uniform() for _ in range(3)] == [0.2706129375647399, 0.6189835150824522, 0.038714373390908996]


def test_philox_restatement_matches_reference_streams():
    g = _load("philox.npz")
    for seed, key, draws in zip(g["seeds"], g["keys"], g["draws"]):
        r = OracleRng(int(seed))
        assert r.key == [int(key[0]), int(key[1])]
        assert [r.uniform() for _ in range(draws.size)] == draws.tolist()


def test_spawned_streams_match_reference():
    g = _load("philox.npz")
    for seed, sk, key, draws in zip(g["spawn_seeds"], g["spawn_keys_flat"], g["spawn_philox_keys"],
                                    g["spawn_draws"]):
        spawn = tuple(int(v) for v in sk.strip("()").split(",") if v.strip())
        assert seedseq_state_u64(int(seed), spawn) == [int(key[0]), int(key[1])]
        r = OracleRng(int(seed), spawn)
        assert [r.uniform() for _ in range(draws.size)] == draws.tolist()


def _blocks(arr):
    return [np.asarray(b, dtype=np.int64) for b in arr]


def case_matrix(g):
    """Dense array, or the CSR matrix for the sparse cases."""
    if "a_indptr" in g.files:
        import scipy.sparse as sp

        return sp.csr_matrix((g["a_data"], g["a_indices"], g["a_indptr"]), shape=tuple(g["a_shape"]))
    return g["a"]


def _oracle_for(g):
    algo = str(g["algorithm"])
    col = _blocks(g["col_blocks"]) if "col_blocks" in g.files else None
    return OracleSolver(case_matrix(g), g["b"], _blocks(g["row_blocks"]), col, float(g["alpha"]), algo)


CASES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLD, "case_*.npz")))


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference_case(case):
    g = _load(case)
    orc = _oracle_for(g)
    assert np.array_equal(orc.row_sampler.cumulative, g["row_cum"])
    assert orc.row_scales == g["row_scales"].tolist()
    if orc.extended:
        assert np.array_equal(orc.col_sampler.cumulative, g["col_cum"])
    z0 = g["z0"] if "z0" in g.files else None
    res = orc.run(int(g["seed"]), int(g["max_iters"]), float(g["tol"]), g["x_star"], int(g["stride"]),
                  str(g["mode"]), z0=z0, record=True)
    assert res["iters"] == int(g["iters"])
    assert res["converged"] == bool(g["converged"])
    if str(g["mode"]) != "max_iters_only":
        assert res["final_error"] == pytest.approx(float(g["final_error"]), rel=1e-9, abs=1e-15)
        assert np.array_equal(res["checkpoints"], g["checkpoints"])
        np.testing.assert_allclose(res["errors"], g["errors"], rtol=1e-9, atol=1e-15)
    npk = min(len(res["picks"]), len(g["picks"]))
    assert np.array_equal(res["picks"][:npk], g["picks"][:npk])
    # per-step snapshots
    x = np.zeros(case_matrix(g).shape[1])
    z = (g["b"].copy() if z0 is None else np.array(z0)) if orc.extended else None
    picks = orc.picks(OracleRng(int(g["seed"])), int(max(g["ks"])))
    for k in range(1, int(max(g["ks"])) + 1):
        orc.step(x, z, int(picks[k - 1, 0]), int(picks[k - 1, 1]))
        if k in set(g["ks"].tolist()):
            np.testing.assert_allclose(x, g[f"x_{k}"], rtol=1e-12, atol=1e-14)
            if z is not None:
                np.testing.assert_allclose(z, g[f"z_{k}"], rtol=1e-12, atol=1e-14)


def test_oracle_c1_against_reference_run():
    """C1 (2000x500, blocks 100/100, alpha = 1/beta_max, seed 17) to
    ||x - x*|| <= 1e-6 ||x*||: same ITER, same block sequence, same iterates."""
    from paper_2001_04179_b200.workloads import c1_matrix

    g = _load("c1_golden.npz")
    a = c1_matrix()
    ptr = np.arange(0, 2001, 100)
    cptr = np.arange(0, 501, 100)
    orc = OracleSolver(a, g["b"], ptr, cptr, float(g["alpha"]), "rebk")
    assert np.array_equal(orc.row_sampler.cumulative, g["row_cum"])
    assert np.array_equal(orc.col_sampler.cumulative, g["col_cum"])
    res = orc.run(int(g["seed"]), 50_000, float(g["tol"]), g["x_star"])
    assert res["iters"] == int(g["iters"])
    assert np.array_equal(res["picks"], g["picks"].astype(np.int64))
    k = int(g["iters"])
    rel = np.linalg.norm(res["x"] - g[f"x_{k}"]) / np.linalg.norm(g[f"x_{k}"])
    assert rel <= 1e-12
    relz = np.linalg.norm(res["z"] - g[f"z_{k}"]) / np.linalg.norm(g[f"z_{k}"])
    assert relz <= 1e-12


@pytest.mark.slow
def test_oracle_c4_against_reference_run():
    """C4 (sparse 200000 x 50000, 1e7 nnz, blocks 2000/1000): same ITER,
    same block sequence, same iterates as the reference."""
    if not os.path.exists(os.path.join(GOLD, "c4_golden.npz")):
        pytest.skip("c4 golden vectors not generated")
    from paper_2001_04179_b200.workloads import c4_matrix

    g = _load("c4_golden.npz")
    s, _ = c4_matrix()
    orc = OracleSolver(s, g["b"], np.arange(0, 200001, 2000), np.arange(0, 50001, 1000), float(g["alpha"]))
    assert np.array_equal(orc.row_sampler.cumulative, g["row_cum"])
    assert np.array_equal(orc.col_sampler.cumulative, g["col_cum"])
    res = orc.run(int(g["seed"]), 50_000, float(g["tol"]), g["x_star"], rng=None)
    assert res["iters"] == int(g["iters"])
    assert np.array_equal(res["picks"], g["picks"].astype(np.int64))
    k = int(g["iters"])
    assert np.linalg.norm(res["x"] - g[f"x_{k}"]) <= 1e-12 * np.linalg.norm(g[f"x_{k}"])
    assert np.linalg.norm(res["z"] - g[f"z_{k}"]) <= 1e-12 * np.linalg.norm(g[f"z_{k}"])


def test_oracle_multi_rhs_mini_columns():
    """Config-5 family at 6000 x 600 with 8 RHS: each column is one
    single-RHS REBK run on the fp64 upcast; the oracle reproduces two of the
    reference's per-column ITER."""
    from paper_2001_04179_b200.workloads import c5_arrays

    g = _load("c5mini_golden.npz")
    a32, b32, xs = c5_arrays(6000, 600, 8)
    a = a32.astype(np.float64)
    for c in (0, 1):
        orc = OracleSolver(a, b32[:, c].astype(np.float64), np.r_[np.arange(0, 6000, 64), 6000],
                           np.r_[np.arange(0, 600, 64), 600], float(g["alpha"]))
        res = orc.run(17, 50_000, float(g["tols"][c]), xs[:, c])
        assert res["iters"] == int(g["iters"][c])

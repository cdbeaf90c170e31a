"""The native MatrixMarket reader (librebk rebk_mm_read, csrc/rebk_mmio.cpp)
against the reference reader (kaczmarz.matrix_io, matrix_io.py:67-222) on
committed fixtures: the same CSR arrays (or dense array) bit for bit, the
same error text and line number for every malformed file
(tests/golden/gen_mm.py recorded the reference's answers).  Host only."""

import os

import numpy as np
import pytest

from paper_2001_04179_b200 import matrix_io as MI

MM = os.path.join(os.path.dirname(__file__), "golden", "mm")
EXP = np.load(os.path.join(MM, "mm_expected.npz"))
FILES = sorted(f for f in os.listdir(MM) if not f.endswith(".npz"))


@pytest.mark.parametrize("name", FILES)
def test_reader_matches_reference(name):
    key = name.replace(".", "_")
    path = os.path.join(MM, name)
    if key + "__error" in EXP.files:
        msg, line = EXP[key + "__error"]
        with pytest.raises(MI.MatrixMarketError) as info:
            MI.read_vector(path) if name.startswith("vec_") else MI.read_matrix_market(path)
        assert info.value.lineno == int(line)
        assert str(info.value) == f"{path}:{line}: {msg}"
        return
    if name.startswith("vec_"):
        np.testing.assert_array_equal(MI.read_vector(path), EXP[key + "__vec"])
        return
    m = MI.read_matrix_market(path)
    if key + "__dense" in EXP.files:
        assert not m.is_sparse
        np.testing.assert_array_equal(m.to_dense(), EXP[key + "__dense"])
    else:
        assert m.is_sparse
        c = m._csr
        assert tuple(c.shape) == tuple(EXP[key + "__shape"])
        np.testing.assert_array_equal(c.indptr, EXP[key + "__indptr"])
        np.testing.assert_array_equal(c.indices, EXP[key + "__indices"])
        np.testing.assert_array_equal(c.data, EXP[key + "__data"])


@pytest.mark.filterwarnings("ignore::DeprecationWarning")
def test_round_trip_and_threads(tmp_path):
    """write -> read round trip at full precision; a file large enough for
    the multithreaded parse gives the same arrays as scipy's own reader."""
    import scipy.io
    import scipy.sparse as sp

    g = np.random.default_rng(3)
    s = sp.random(3000, 2000, density=0.01, format="csr", random_state=g, data_rvs=g.standard_normal)
    a = MI.Matrix.from_sparse(s)
    p = tmp_path / "big.mtx"
    MI.write_matrix_market(a, p)
    b = MI.read_matrix_market(p)
    ref = sp.csr_matrix(scipy.io.mmread(str(p)))
    ref.sort_indices()
    np.testing.assert_array_equal(b._csr.indptr, ref.indptr)
    np.testing.assert_array_equal(b._csr.indices, ref.indices)
    np.testing.assert_array_equal(b._csr.data, ref.data)
    v = g.standard_normal(17)
    MI.write_vector(v, tmp_path / "v.txt")
    np.testing.assert_array_equal(MI.read_vector(tmp_path / "v.txt"), v)


def test_missing_file():
    with pytest.raises(FileNotFoundError):
        MI.load_suitesparse("/nonexistent/abtaha1.mtx")

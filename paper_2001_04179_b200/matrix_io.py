"""MatrixMarket files in and out, with the native reader.

Same surface as the reference's ``kaczmarz.matrix_io`` (matrix_io.py):
``read_matrix_market`` / ``read_vector`` / ``write_matrix_market`` /
``write_vector`` / ``load_suitesparse`` and ``MatrixMarketError`` (a
ValueError carrying path and line).  The matrix reader is librebk's
multithreaded C++ parser (``rebk_mm_read``, csrc/rebk_mmio.cpp): it applies
the reference's acceptance rules and error texts and hands back the CSR
arrays (sorted columns, duplicates summed, explicit zeros dropped) that
``rebk_ctx_create_csr`` consumes, or a dense array above the density
threshold.  SuiteSparse matrices (the paper's Table 3) load through the same
path when a file is supplied; none ship with this repo.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import scipy.sparse as sp

from . import _lib
from .matrix import Matrix

DENSE_DENSITY_THRESHOLD = 0.05
_BANNER = "%%matrixmarket"
_HOST_THREADS = min(16, os.cpu_count() or 1)


class MatrixMarketError(ValueError):
    """Malformed MatrixMarket content, with file and line context."""

    def __init__(self, path, lineno: int, message: str):
        super().__init__(f"{path}:{lineno}: {message}")
        self.path = path
        self.lineno = lineno


def read_matrix_market(path, dense_threshold: float = DENSE_DENSITY_THRESHOLD) -> Matrix:
    """Load a real matrix from a MatrixMarket file (native parser)."""
    lib = _lib.load()
    out = _lib.RebkMmMatrix()
    rc = lib.rebk_mm_read(os.fsencode(path), float(dense_threshold), _HOST_THREADS, ctypes.byref(out))
    if rc != _lib.REBK_OK:
        msg = lib.rebk_last_error().decode(errors="replace")
        if out.err_line == 0 and msg.startswith(("cannot open", "read error")):
            raise FileNotFoundError(path) if msg.startswith("cannot open") else OSError(msg)
        raise MatrixMarketError(path, int(out.err_line), msg)
    try:
        m, n = int(out.rows), int(out.cols)
        if out.dense:
            dense = np.ctypeslib.as_array(out.values, shape=(m * n,)).reshape(m, n).copy()
            return Matrix.from_dense(dense)
        nnz = int(out.nnz)
        indptr = np.ctypeslib.as_array(out.indptr, shape=(m + 1,)).copy()
        indices = np.ctypeslib.as_array(out.indices, shape=(max(nnz, 1),))[:nnz].copy()
        data = np.ctypeslib.as_array(out.values, shape=(max(nnz, 1),))[:nnz].copy()
        return Matrix.from_sparse(sp.csr_matrix((data, indices, indptr), shape=(m, n)))
    finally:
        lib.rebk_mm_free(ctypes.byref(out))


def _parse_value(path, lineno, token) -> float:
    try:
        value = float(token)
    except ValueError:
        raise MatrixMarketError(path, lineno, f"not a number: {token!r}") from None
    if not np.isfinite(value):
        raise MatrixMarketError(path, lineno, f"non-finite value: {token!r}")
    return value


def read_vector(path) -> np.ndarray:
    """A vector file: a one-column MatrixMarket array, or one value per line
    ('%' / '#' comments and blank lines skipped) (matrix_io.py:180-210)."""
    with open(path, "r", encoding="ascii") as handle:
        lines = handle.read().splitlines()
    if not lines:
        raise MatrixMarketError(path, 1, "empty file")
    if lines[0].strip().lower().startswith(_BANNER):
        head = lines[0].strip().lower().split()
        if len(head) != 5 or head[1] != "matrix":
            raise MatrixMarketError(path, 1, "malformed banner; expected '%%MatrixMarket matrix ...'")
        if head[2] not in ("coordinate", "array"):
            raise MatrixMarketError(path, 1, f"unsupported format {head[2]!r}")
        if head[3] not in ("real", "integer", "pattern"):
            raise MatrixMarketError(path, 1, f"unsupported field {head[3]!r}")
        if head[4] not in ("general", "symmetric"):
            raise MatrixMarketError(path, 1, f"unsupported symmetry {head[4]!r}")
        if head[2] != "array" or head[3] == "pattern":
            raise MatrixMarketError(path, 1, "vector files must be array format with values")
        body = [(no, ln.strip()) for no, ln in enumerate(lines[1:], start=2)
                if ln.strip() and not ln.strip().startswith("%")]
        size_no, size_line = body[0] if body else (len(lines), "")
        tokens = size_line.split()
        if len(tokens) != 2 or not all(t.isdigit() for t in tokens):
            raise MatrixMarketError(path, size_no, f"malformed size line: {size_line!r}")
        rows, cols = int(tokens[0]), int(tokens[1])
        if cols != 1:
            raise MatrixMarketError(path, size_no, "vector files must have one column")
        values = [_parse_value(path, no, ln.split()[0]) for no, ln in body[1:]]
        if len(values) != rows:
            raise MatrixMarketError(path, len(lines), f"expected {rows} values, got {len(values)}")
        return np.asarray(values)
    values = [_parse_value(path, no, ln.strip()) for no, ln in enumerate(lines, start=1)
              if ln.strip() and not ln.strip().startswith(("%", "#"))]
    if not values:
        raise MatrixMarketError(path, len(lines), "no values found")
    return np.asarray(values)


def write_matrix_market(m: Matrix, path) -> None:
    """coordinate / real / general, every value at round-trip precision."""
    if m.is_sparse:
        coo = m._csr.tocoo()
        rows, cols, vals = coo.row, coo.col, coo.data
    else:
        d = m.to_dense()
        rows, cols = np.nonzero(d)
        vals = d[rows, cols]
    with open(path, "w", encoding="ascii") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{m.rows} {m.cols} {len(vals)}\n")
        fh.writelines(f"{i + 1} {j + 1} {float(v)!r}\n" for i, j, v in zip(rows, cols, vals))


def write_vector(v: np.ndarray, path) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.writelines(f"{float(x)!r}\n" for x in np.asarray(v, dtype=np.float64))


def load_suitesparse(path) -> Matrix:
    """A SuiteSparse matrix from a supplied .mtx path (no download)."""
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    return read_matrix_market(path)

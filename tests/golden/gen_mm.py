"""MatrixMarket fixtures and the REFERENCE reader's results on them.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_mm.py

Writes small .mtx / vector files under tests/golden/mm/ (seeded synthetic
content covering the format's branches and its error cases) and records what
kaczmarz.matrix_io.read_matrix_market / read_vector return or raise
(mm_expected.npz).  Runs only where the reference is importable; the files
it writes are committed."""

import os
import sys

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mm")
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")
from kaczmarz import matrix_io as MI  # noqa: E402


def w(name, text):
    with open(os.path.join(HERE, name), "w", encoding="ascii") as fh:
        fh.write(text)


def files():
    g = np.random.default_rng(7)
    # sparse general real, comments / blank lines, a duplicate pair, an explicit zero
    m, n = 40, 30
    ent = []
    for _ in range(50):
        ent.append((int(g.integers(1, m + 1)), int(g.integers(1, n + 1)), float(g.standard_normal())))
    ent.append(ent[3][:2] + (0.25,))  # duplicate of entry 3
    ent.append((m, n, 0.0))           # explicit zero
    lines = [f"{i} {j} {v!r}\n" if k % 7 else f"  {i}\t{j}   {v!r}  \n" for k, (i, j, v) in enumerate(ent)]
    h = len(lines) // 2
    w("sparse_general.mtx", "%%MatrixMarket matrix coordinate real general\n% a comment\n\n"
      f"{m} {n} {len(ent)}\n" + "".join(lines[:h]) + "% mid comment\n\n" + "".join(lines[h:]))
    # symmetric (lower triangle), integer field
    ent = [(i, j, int(g.integers(-5, 6))) for i in range(1, 21) for j in range(1, i + 1) if g.random() < 0.08]
    w("sym_integer.mtx", "%%MatrixMarket matrix coordinate integer symmetric\n"
      f"20 20 {len(ent)}\n" + "".join(f"{i} {j} {v}\n" for i, j, v in ent))
    # pattern
    ent = sorted({(int(g.integers(1, 51)), int(g.integers(1, 41))) for _ in range(60)})
    w("pattern.mtx", "%%MatrixMarket matrix coordinate pattern general\n"
      f"50 40 {len(ent)}\n" + "".join(f"{i} {j}\n" for i, j in ent))
    # dense enough to load dense (>= 5% distinct)
    ent = [(i, j, float(g.standard_normal())) for i in range(1, 9) for j in range(1, 7) if g.random() < 0.5]
    w("dense_coord.mtx", "%%MatrixMarket matrix coordinate real general\n"
      f"8 6 {len(ent)}\n" + "".join(f"{i} {j} {v!r}\n" for i, j, v in ent))
    # Python float / int grammar: signs, exponents, underscores, leading '+', uppercase banner
    w("grammar.mtx", "%%MATRIXMARKET Matrix Coordinate Real General\n"
      "100 100 6\n+1 1 1e3\n2 +2 -2.5E-3\n3 3 .5\n4 4 5.\n1_0 1_1 1_000.000_1\n0007 8 +0.0625\n")
    # array general / symmetric
    vals = [float(v) for v in g.standard_normal(12)]
    w("array_general.mtx", "%%MatrixMarket matrix array real general\n4 3\n"
      + "".join(f"{v!r}\n" for v in vals[:6]) + "% c\n" + " ".join(repr(v) for v in vals[6:]) + "\n")
    vals = [float(v) for v in g.standard_normal(10)]
    w("array_sym.mtx", "%%MatrixMarket matrix array real symmetric\n4 4\n" + "".join(f"{v!r}\n" for v in vals))
    # vectors
    w("vec_plain.txt", "# x\n1.5\n\n-2.25\n% y\n3e-2\n")
    w("vec_mm.mtx", "%%MatrixMarket matrix array real general\n3 1\n1.0\n2.0\n-3.5\n")
    # errors
    w("err_banner.mtx", "%%MatrixMarket tensor coordinate real general\n2 2 0\n")
    w("err_format.mtx", "%%MatrixMarket matrix sparse real general\n2 2 0\n")
    w("err_field.mtx", "%%MatrixMarket matrix coordinate complex general\n2 2 0\n")
    w("err_sym.mtx", "%%MatrixMarket matrix coordinate real hermitian\n2 2 0\n")
    w("err_nosize.mtx", "%%MatrixMarket matrix coordinate real general\n% only comments\n\n")
    w("err_size.mtx", "%%MatrixMarket matrix coordinate real general\n2 2\n1 1 1.0\n")
    w("err_dims.mtx", "%%MatrixMarket matrix coordinate real general\n0 2 0\n")
    w("err_fields.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n2 2\n")
    w("err_index.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n2.0 2 1.0\n")
    w("err_bounds.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n4 2 1.0\n")
    w("err_nan.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n2 2 nan\n")
    w("err_number.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n2 2 1.2.3\n")
    w("err_upper.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n1 1 1.0\n1 2 1.0\n")
    w("err_count.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1.0\n2 2 1.0\n\n")
    w("err_array_count.mtx", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n")
    w("err_array_sym.mtx", "%%MatrixMarket matrix array real symmetric\n2 3\n1\n2\n3\n")
    w("err_empty.mtx", "")


def main():
    os.makedirs(HERE, exist_ok=True)
    files()
    out = {}
    for name in sorted(os.listdir(HERE)):
        path = os.path.join(HERE, name)
        key = name.replace(".", "_")
        try:
            if name.startswith("vec_"):
                out[key + "__vec"] = MI.read_vector(path)
                continue
            m = MI.read_matrix_market(path)
            if m.is_sparse:
                c = m._csr
                out[key + "__indptr"] = c.indptr.astype(np.int64)
                out[key + "__indices"] = c.indices.astype(np.int32)
                out[key + "__data"] = c.data
                out[key + "__shape"] = np.asarray(c.shape)
            else:
                out[key + "__dense"] = m.to_dense()
        except MI.MatrixMarketError as exc:
            out[key + "__error"] = np.asarray([str(exc).split(": ", 1)[1], str(exc.lineno)])
            print(f"{name}: {exc}")
    np.savez_compressed(os.path.join(HERE, "mm_expected.npz"), **out)
    print(f"{len(out)} entries")


if __name__ == "__main__":
    main()

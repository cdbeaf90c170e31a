"""The reference's generators on small shapes (problems.py:60-127 with its
Jacobi-SVD oracle), recorded for tests/test_generators.py.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_generators.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
if "/root/reference/pkg/src" not in sys.path:
    sys.path.insert(0, "/root/reference/pkg/src")
import kaczmarz as K  # noqa: E402

CASES = [
    # name, kind, (m, n, r, kappa) / (m, n), matrix seed, rhs seed, inconsistent, perp_scale
    ("t1_tall", 1, (60, 25, 20, 3.0), 11, 12, True, 1.0),
    ("t1_wide", 1, (30, 70, 18, 10.0), 13, 14, True, 0.5),
    ("t1_consistent", 1, (40, 30, 30, 2.0), 15, 16, False, 1.0),
    ("t2_tall", 2, (80, 35), 17, 18, True, 2.0),
    ("t2_wide", 2, (25, 50), 19, 20, False, 1.0),
]


def main():
    out = {}
    for name, kind, shape, ms, rs, inc, ps in CASES:
        a = K.gen_type1(*shape, seed=ms) if kind == 1 else K.gen_type2(*shape, seed=ms)
        p = K.make_rhs(a, seed=rs, inconsistent=inc, perp_scale=ps, kappa_bound=shape[3] if kind == 1 else None)
        out[f"{name}__a"] = a.to_dense()
        out[f"{name}__b"] = p.b
        out[f"{name}__x_star"] = p.x_star
        out[f"{name}__b_perp"] = p.b_perp
        out[f"{name}__meta"] = np.asarray([p.meta.declared_rank, float(p.meta.consistent), p.meta.residual_norm])
        print(name, p.meta)
    # full row rank + inconsistent must raise
    try:
        K.make_rhs(K.gen_type2(20, 30, seed=3), seed=4, inconsistent=True)
    except ValueError as exc:
        out["err_full_row_rank"] = np.asarray(str(exc))
    np.savez_compressed(os.path.join(HERE, "generators.npz"), **out)


if __name__ == "__main__":
    main()

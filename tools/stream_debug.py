"""Find which shape feature breaks the streaming kernel (GPU box)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["REBK_NO_FAST"] = "1"
os.environ["REBK_STREAM"] = "2"
import paper_2001_04179_b200 as P  # noqa: E402


def trial(m, n, tr, tc, grid=0, alg="rebk"):
    if grid:
        os.environ["REBK_GRID"] = str(grid)
    else:
        os.environ.pop("REBK_GRID", None)
    rs = np.random.default_rng(5)
    a = rs.standard_normal((m, n))
    b = a @ rs.standard_normal(n)
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=np.zeros(n), b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    cfg = P.SolverConfig(algorithm=alg, alpha=0.5, seed=3, max_iters=20,
                         row_partition=P.contiguous_partition(m, tr, "row"),
                         col_partition=P.contiguous_partition(n, tc, "col"),
                         stop=P.StoppingRule(mode="max_iters_only"), beta_max=1.0)
    try:
        t = P.run(prob, cfg)
        print(f"m={m} n={n} tr={tr} tc={tc} grid={grid}: ok path={t.kernel_path} grid={t.grid_ctas}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"m={m} n={n} tr={tr} tc={tc} grid={grid}: FAIL {e}", flush=True)
        sys.exit(1)


for args in [(701, 334, 100, 60), (701, 334, 97, 60), (701, 334, 100, 61), (700, 333, 100, 60), (701, 333, 97, 61),
             (2000, 500, 100, 100, 4)]:
    trial(*args)

"""Small runs of every kernel family for compute-sanitizer (one tool per
gpurun call; B200_PROFILING.md): the split / fused clustered dense kernels
(C1), the streaming kernel (forced), the row-sharded kernel with 2 emulated
ranks, the CSR kernel, the general kernel (DSBGS), the multi-RHS tcgen05
kernel and device beta.  Each case runs a few dozen iterations.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2001_04179_b200 as P  # noqa: E402
from paper_2001_04179_b200 import _lib  # noqa: E402

ITERS = int(os.environ.get("SAN_ITERS", "20"))


def dense(m, n, seed):
    g = np.random.default_rng(seed)
    a = g.standard_normal((m, n))
    xs = g.standard_normal(n)
    b = a @ xs + 0.05 * g.standard_normal(m)
    return P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=np.linalg.lstsq(a, b, rcond=None)[0], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))


def cfg(m, n, tr, tc, algo="rebk", iters=ITERS):
    kw = dict(algorithm=algo, alpha=1.0, seed=3, max_iters=iters, row_partition=P.contiguous_partition(m, tr, "row"),
              stop=P.StoppingRule(tol=1e-12), beta_max=0.3)
    if algo in ("rebk", "dsbgs"):
        kw["col_partition"] = P.contiguous_partition(n, tc, "col")
    return P.SolverConfig(**kw)


def main():
    out = []
    p = dense(2000, 500, 1)
    t = P.run(p, cfg(2000, 500, 100, 100))
    out.append(f"split/fused dense (C1 shape): path {t.kernel_path}, {t.iters} iters")
    os.environ["REBK_SPLIT"] = "0"
    t = P.run(p, cfg(2000, 500, 100, 100))
    out.append(f"fused clustered dense: path {t.kernel_path}")
    os.environ["REBK_SPLIT"] = "1"
    os.environ["REBK_STREAM"] = "2"
    os.environ["REBK_NO_FAST"] = "1"
    t = P.run(p, cfg(2000, 500, 100, 100))
    out.append(f"streaming dense (forced): path {t.kernel_path}")
    del os.environ["REBK_STREAM"], os.environ["REBK_NO_FAST"]
    t = P.run(p, cfg(2000, 500, 100, 100, algo="dsbgs"))
    out.append(f"general dense (dsbgs): path {t.kernel_path}")
    from paper_2001_04179_b200.sharded import run_persistent_virtual

    ctx = P.prepare(p, cfg(2000, 500, 100, 100))
    c = ctx.make_cfg(stop_mode="oracle_error", tol=1e-12, stride=1, max_iters=ITERS, key=_lib.philox_key(3))
    r = run_persistent_virtual(p.a.to_dense(), p.b, p.x_star, c, ctx._row_ptr, 2)
    out.append(f"row-sharded persistent, 2 emulated ranks: path {r['kernel_path']}")
    import scipy.sparse as sp

    g = np.random.default_rng(2)
    s = sp.random(3000, 800, density=0.01, format="csr", random_state=g)
    s.data = g.standard_normal(s.nnz)
    ps = P.ProblemInstance(a=P.Matrix.from_sparse(s), b=s @ g.standard_normal(800), x_star=g.standard_normal(800),
                           b_perp=None, meta=P.ProblemMeta(0, None, False, 0, 0.0))
    t = P.run(ps, cfg(3000, 800, 100, 50))
    out.append(f"CSR: path {t.kernel_path}")
    from paper_2001_04179_b200.multirhs import run_multi
    from paper_2001_04179_b200.workloads import c5_arrays

    a32, b32, xs = c5_arrays(2000, 400, 8)
    t5 = run_multi(a32, b32, P.SolverConfig(algorithm="rebk", alpha=20.0, seed=17, max_iters=ITERS,
                                            row_partition=P.contiguous_partition(2000, 64, "row"),
                                            col_partition=P.contiguous_partition(400, 64, "col"),
                                            stop=P.StoppingRule(mode="max_iters_only"), beta_max=0.02))
    out.append(f"multi-RHS tcgen05: path {t5.kernel_path}")
    b = P.device_beta_max(p.a, P.contiguous_partition(2000, 100, "row"), P.contiguous_partition(500, 100, "col"))
    out.append(f"device beta {b[2]:.6g}")
    print("\n".join(out))


if __name__ == "__main__":
    main()

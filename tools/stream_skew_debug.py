"""Debug: streaming kernel vs golden snapshots / the general kernel at small iteration counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["REBK_NO_FAST"] = "1"
import numpy as np
import paper_2001_04179_b200 as P
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import c1_instance, rel

g, a, prob, cfg = c1_instance()
for K in (1, 2, 3, 10, 100):
    out = {}
    for mode in ("2", "0"):
        os.environ["REBK_STREAM"] = mode
        c = P.SolverConfig(algorithm="rebk", alpha=cfg.alpha, seed=cfg.seed, max_iters=K, row_partition=cfg.row_partition,
                           col_partition=cfg.col_partition, stop=P.StoppingRule(mode="max_iters_only"), beta_max=cfg.beta_max)
        t = P.run(prob, c)
        out[mode] = t
    s, v = out["2"], out["0"]
    msg = f"K={K} paths {s.kernel_path}/{v.kernel_path} x rel {rel(s.x, v.x):.2e} z rel {rel(s.z, v.z):.2e}"
    if f"x_{K}" in g.files:
        msg += f" | vs golden: stream x {rel(s.x, g[f'x_{K}']):.2e} z {rel(s.z, g[f'z_{K}']):.2e}; general x {rel(v.x, g[f'x_{K}']):.2e}"
    print(msg)
os.environ["REBK_STREAM"] = "2"
t = P.run(prob, cfg)
k = int(g["iters"])
print("full run iters", t.iters, k, "x", rel(t.x, g[f"x_{k}"]), "z", rel(t.z, g[f"z_{k}"]))

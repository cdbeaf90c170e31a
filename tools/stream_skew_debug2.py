import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["REBK_NO_FAST"] = "1"
import numpy as np
import paper_2001_04179_b200 as P
from test_gpu_parity import c1_instance, rel
g, a, prob, cfg = c1_instance()
def run(K, stream, **env):
    os.environ["REBK_STREAM"] = stream
    for k, v in env.items(): os.environ[k] = v
    c = P.SolverConfig(algorithm="rebk", alpha=cfg.alpha, seed=cfg.seed, max_iters=K, row_partition=cfg.row_partition,
                       col_partition=cfg.col_partition, stop=P.StoppingRule(mode="max_iters_only"), beta_max=cfg.beta_max)
    t = P.run(prob, c)
    for k in env: del os.environ[k]
    return t
ref = run(2, "0")
for env in ({}, {"REBK_STREAM_DBG": "1"}, {"REBK_GRID": "2"}, {"REBK_GRID": "2", "REBK_STREAM_DBG": "1"}):
    t = run(2, "2", **env)
    print(env, "G", t.grid_ctas, "x", f"{rel(t.x, ref.x):.2e}", "z", f"{rel(t.z, ref.z):.2e}")

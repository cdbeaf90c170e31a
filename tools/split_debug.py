"""Run C2 through the split path with small budgets (debugging aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04179_b200 as P
from paper_2001_04179_b200 import workloads, StoppingRule
wl = workloads.build(sys.argv[1] if len(sys.argv) > 1 else "c2")
for mode, it in [("max_iters_only", 1), ("max_iters_only", 20), ("oracle_error", 20), ("oracle_error", 50000)]:
    cfg = wl.config(max_iters=it)
    if mode == "max_iters_only":
        cfg.stop = StoppingRule(mode="max_iters_only")
    t0 = time.time()
    tr = P.run(wl.problem, cfg)
    print(mode, it, "->", tr.iters, tr.converged, tr.kernel_path, tr.grid_ctas, f"{tr.wall_time*1e3:.2f} ms", f"{time.time()-t0:.2f}s", flush=True)

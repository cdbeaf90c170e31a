"""Small fast-path run (C1 instance, 60 iterations) for sanitizer / profiler passes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04179_b200 as P
from paper_2001_04179_b200 import workloads
it = int(sys.argv[1]) if len(sys.argv) > 1 else 60
wl = workloads.build("c1")
cfg = wl.config(max_iters=it)
tr = P.run(wl.problem, cfg)
print("iters", tr.iters, "path", tr.kernel_path, "grid", tr.grid_ctas, "err", tr.final_error)

"""Where the per-solve fixed cost of the public run() path goes (C1):
device copy of A, the device run itself, release.  usage: python tools/e2e_overhead.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04179_b200 as P  # noqa: E402
from paper_2001_04179_b200 import workloads  # noqa: E402

wl = workloads.build(sys.argv[1] if len(sys.argv) > 1 else "c1")
if "--torch" in sys.argv:
    # bench.py conditions: torch owns a CUDA context and memory, A lives in pinned host memory
    import torch

    keep = torch.empty(wl.problem.a.shape, dtype=torch.float64, device="cuda")
    a_pin = torch.from_numpy(wl.problem.a.to_dense()).pin_memory()
    wl.problem = P.ProblemInstance(a=P.Matrix.from_dense(a_pin.numpy()), b=wl.problem.b, x_star=wl.problem.x_star,
                                   b_perp=None, meta=wl.problem.meta)
for mi in (1, 50_000):
    cfg = wl.config(max_iters=mi)
    for rep in range(4):
        t0 = time.perf_counter()
        ctx = P.prepare(wl.problem, cfg)
        t1 = time.perf_counter()
        dm = ctx.device_matrix
        t2 = time.perf_counter()
        tr = P.run(wl.problem, cfg)
        t3 = time.perf_counter()
        wl.problem.a.release_device()
        t4 = time.perf_counter()
        print(f"max_iters={mi} rep {rep}: prepare {1e3*(t1-t0):.1f} ms, device copy {1e3*(t2-t1):.1f} ms, "
              f"run() {1e3*(t3-t2):.1f} ms (loop {1e3*tr.wall_time:.1f} ms, iters {tr.iters}), "
              f"release {1e3*(t4-t3):.1f} ms", flush=True)

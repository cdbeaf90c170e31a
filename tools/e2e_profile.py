"""cProfile of one public run() on a workload with A in pinned host memory and
the device copy released first (bench.py's e2e conditions).
usage: python tools/e2e_profile.py [c2]"""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04179_b200 as P  # noqa: E402
from paper_2001_04179_b200 import workloads  # noqa: E402

wl = workloads.build(sys.argv[1] if len(sys.argv) > 1 else "c2")
if wl.problem.a.is_sparse:
    mat = wl.problem.a
else:
    a_pin = torch.from_numpy(wl.problem.a.to_dense()).pin_memory()
    mat = P.Matrix.from_dense(a_pin.numpy())
prob = P.ProblemInstance(a=mat, b=wl.problem.b, x_star=wl.problem.x_star, b_perp=None, meta=wl.problem.meta)
cfg = wl.config()
cfg.row_partition, cfg.col_partition = wl.row_partition, wl.col_partition
for _ in range(2):
    P.run(prob, cfg)
    prob.a.release_device()
import time  # noqa: E402

for _ in range(4):
    t0 = time.perf_counter()
    tr = P.run(prob, cfg)
    t1 = time.perf_counter()
    prob.a.release_device()
    t2 = time.perf_counter()
    ctx = P.prepare(prob, cfg)
    t3 = time.perf_counter()
    ctx.device_matrix
    t4 = time.perf_counter()
    prob.a.release_device()
    t5 = time.perf_counter()
    print(f"run {1e3*(t1-t0):.1f} ms (loop {tr.wall_time*1e3:.1f}) release {1e3*(t2-t1):.1f} | "
          f"prepare {1e3*(t3-t2):.1f} upload {1e3*(t4-t3):.1f} release {1e3*(t5-t4):.1f}")
if "--cprofile" in sys.argv:
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        tr = P.run(prob, cfg)
        prob.a.release_device()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)

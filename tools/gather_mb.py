"""Host-side sampler weights at C2 (4000 x 10000, 50 column blocks of 200):
librebk's gather pass at several thread counts, then the 50 numpy dots.
usage: python tools/gather_mb.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_04179_b200 import _lib  # noqa: E402

A = np.random.default_rng(0).standard_normal((4000, 10000))
lib = _lib.load()
buf = np.empty(A.size)
ptr = np.arange(0, 10001, 200, dtype=np.int64)
print("cpus", os.cpu_count())
for nt in (1, 4, 8, 16, 32):
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        lib.rebk_host_gather_col_blocks(_lib.dptr(A), 4000, 10000, 10000, 50, _lib.i64ptr(ptr), _lib.dptr(buf), nt)
        ts.append(round((time.perf_counter() - t) * 1e3, 2))
    print("gather threads", nt, "ms", ts)
for _ in range(3):
    t = time.perf_counter()
    w = [float(buf[4000 * ptr[k]:4000 * ptr[k + 1]] @ buf[4000 * ptr[k]:4000 * ptr[k + 1]]) for k in range(50)]
    t2 = time.perf_counter()
    w2 = [float(np.ravel(A[:, j:j + 200]) @ np.ravel(A[:, j:j + 200])) for j in range(0, 10000, 200)]
    t3 = time.perf_counter()
    big = float(np.ravel(A) @ np.ravel(A))
    t4 = time.perf_counter()
    print("50 dots ms", round((t2 - t) * 1e3, 2), "ravel+dot ms", round((t3 - t2) * 1e3, 2),
          "one 320MB dot ms", round((t4 - t3) * 1e3, 2), "equal", w == w2)

# bench.py's e2e conditions: A in torch pinned host memory
import torch  # noqa: E402

Ap = torch.from_numpy(A).pin_memory().numpy()
for nt in (8, 16):
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        lib.rebk_host_gather_col_blocks(_lib.dptr(Ap), 4000, 10000, 10000, 50, _lib.i64ptr(ptr), _lib.dptr(buf), nt)
        ts.append(round((time.perf_counter() - t) * 1e3, 2))
    print("pinned A: gather threads", nt, "ms", ts)
for _ in range(3):
    t = time.perf_counter()
    w = [float(buf[4000 * ptr[k]:4000 * ptr[k + 1]] @ buf[4000 * ptr[k]:4000 * ptr[k + 1]]) for k in range(50)]
    print("pinned A: 50 dots ms", round((time.perf_counter() - t) * 1e3, 2))
x = torch.empty(1, device="cuda")  # a live CUDA context, as in the bench
for nt in (8, 16):
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        lib.rebk_host_gather_col_blocks(_lib.dptr(Ap), 4000, 10000, 10000, 50, _lib.i64ptr(ptr), _lib.dptr(buf), nt)
        ts.append(round((time.perf_counter() - t) * 1e3, 2))
    print("pinned A + CUDA ctx: gather threads", nt, "ms", ts)

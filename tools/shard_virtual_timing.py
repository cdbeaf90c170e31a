"""C3 on one B200: the single-GPU streaming kernel against the row-sharded
persistent kernel with P ranks emulated in one launch (each emulated rank
gets 148/P SMs; together they still stream the whole matrix from the one
HBM), so the per-iteration difference is the cost of the in-kernel
cross-rank exchange.  REBK_PROF=1 adds the per-phase breakdown (marks 4 and
12 are the u and dx exchange waits).  Usage: python tools/shard_virtual_timing.py [reps]"""

import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2001_04179_b200 import _lib  # noqa: E402
from paper_2001_04179_b200.matrix import DeviceMatrix  # noqa: E402
from paper_2001_04179_b200.sharded import run_persistent_virtual  # noqa: E402
from paper_2001_04179_b200.workloads import c3_device  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = c3_device()
m, n = wl.shape
tol = wl.rel_tol * float(wl.x_star.norm())
c = wl.cfg("oracle_error", tol, 5000)
dm = DeviceMatrix.from_device_pointer(wl.a.data_ptr(), m, n, n, 0)
x = torch.zeros(n, dtype=torch.float64, device="cuda")
z = torch.empty(m, dtype=torch.float64, device="cuda")
best = 1e9
for _ in range(reps):
    x.zero_()
    z.copy_(wl.b)
    torch.cuda.synchronize()
    tr = _lib.RebkTrace()
    _lib.check(_lib.load().rebk_run_device(dm.handle, ctypes.byref(c), ctypes.c_void_p(wl.b.data_ptr()),
                                           ctypes.c_void_p(wl.x_star.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                           ctypes.c_void_p(z.data_ptr()), None, ctypes.byref(tr)), "run")
    best = min(best, tr.loop_ms)
it1 = int(tr.iters)
print(f"single-GPU stream kernel: ITER {it1}, {best:.2f} ms = {1e3 * best / it1:.1f} us/iter, grid {tr.grid_ctas}",
      flush=True)
xs1 = x.cpu().numpy()
dm.close()
del x, z
for P in (1, 2, 4, 8):
    ms = []
    for _ in range(reps):
        res = run_persistent_virtual(wl.a, wl.b, wl.x_star, c, wl.row_ptr, P)
        ms.append(res["loop_ms"])
    relx = np.linalg.norm(res["x"] - xs1) / np.linalg.norm(xs1)
    print(f"sharded kernel, {P} emulated rank(s) x {res['grid_ctas']} CTAs: ITER {res['iters']}, "
          f"{min(ms):.2f} ms = {1e3 * min(ms) / res['iters']:.1f} us/iter (|dx|/|x| vs single-GPU {relx:.1e})",
          flush=True)

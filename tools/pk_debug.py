"""Compare the persistent multi-RHS kernel with the per-product kernels on
the config-5 mini instance after a few iterations (max_iters_only)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04179_b200 as P  # noqa: E402
from paper_2001_04179_b200.multirhs import run_multi, DeviceMatrix32  # noqa: E402
from paper_2001_04179_b200.workloads import c5_arrays  # noqa: E402

m, n, R, blk = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (6000, 600, 8, 64)))
a32, b32, xs = c5_arrays(m, n, R)
rp, cp = P.contiguous_partition(m, blk, "row"), P.contiguous_partition(n, blk, "col")
a64 = P.Matrix.from_dense(a32.astype(np.float64))
beta = P.compute_beta_max(a64, rp, cp)[2]
dm = DeviceMatrix32(a32)
for its in (1, 2, 3, 5, 20):
    out = {}
    for pk in ("1", "0"):
        os.environ["REBK_MRHS_PK"] = pk
        cfg = P.SolverConfig(algorithm="rebk", alpha=1.0 / beta, seed=17, max_iters=its, row_partition=rp,
                             col_partition=cp, stop=P.StoppingRule(mode="max_iters_only"), beta_max=beta)
        out[pk] = run_multi(a32, b32, cfg, device_matrix=dm, a64=a64)
    dx = np.abs(out["1"].X - out["0"].X).max()
    dz = np.abs(out["1"].Z - out["0"].Z).max()
    print(f"iters={its}: K {out['1'].iters}/{out['0'].iters} max|dX|={dx:.3e} max|dZ|={dz:.3e} "
          f"|X|={np.abs(out['0'].X).max():.3e} nanX={np.isnan(out['1'].X).sum()} nanZ={np.isnan(out['1'].Z).sum()}",
          flush=True)

# where do the two paths differ after one iteration?
out = {}
for pk in ("1", "0"):
    os.environ["REBK_MRHS_PK"] = pk
    cfg = P.SolverConfig(algorithm="rebk", alpha=1.0 / beta, seed=17, max_iters=1, row_partition=rp,
                         col_partition=cp, stop=P.StoppingRule(mode="max_iters_only"), beta_max=beta)
    out[pk] = run_multi(a32, b32, cfg, device_matrix=dm, a64=a64)
dz = np.abs(out["1"].Z - out["0"].Z)
bad_rows = np.where(dz.max(axis=1) > 1e-3)[0]
print("Z bad rows:", len(bad_rows), "tiles:", sorted(set((bad_rows // 128).tolist()))[:60])
print("Z bad cols:", np.where(dz.max(axis=0) > 1e-3)[0].tolist())
z0 = b32
print("Z changed rows (ref):", int((np.abs(out["0"].Z - z0).max(axis=1) > 0).sum()),
      " (pk):", int((np.abs(out["1"].Z - z0).max(axis=1) > 0).sum()))
dx = np.abs(out["1"].X - out["0"].X)
print("X bad rows:", np.where(dx.max(axis=1) > 1e-6)[0][:40].tolist(), "cols", np.where(dx.max(axis=0) > 1e-6)[0].tolist())

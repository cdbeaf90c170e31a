"""CPU restatement of one rank of the row-sharded REBK (TEST INFRASTRUCTURE
ONLY).  Same interface as paper_2001_04179_b200.sharded.CudaShardBackend,
numpy arithmetic; vectors handed to the collective are torch CPU tensors that
share memory with numpy, so a gloo allreduce updates them in place.  Used by
tests/test_sharded_gloo.py to check the sharding logic (row ownership,
which vectors are reduced, the stop rule) against the single-process oracle.
"""

from __future__ import annotations

import numpy as np


class NumpyShardBackend:
    def __init__(self, a_local: np.ndarray, b_local: np.ndarray, x_star: np.ndarray | None, extended: bool):
        import torch

        self.torch = torch
        self.a = np.ascontiguousarray(a_local, dtype=np.float64)
        self.m_local, self.n = self.a.shape
        self.b = np.asarray(b_local, dtype=np.float64)
        self.z = self.b.copy() if extended else None
        self.x = np.zeros(self.n)
        self.xs = x_star
        self.extended = extended

    def colstep(self, c_lo, c_hi):
        u = self.a[:, c_lo:c_hi].T @ self.z if self.m_local else np.zeros(c_hi - c_lo)
        return self.torch.from_numpy(np.ascontiguousarray(u))

    def zupdate(self, c_lo, c_hi, scale, u):
        if self.m_local:
            self.z -= scale * (self.a[:, c_lo:c_hi] @ u.numpy())

    def rowstep(self, lo, hi):
        blk = self.a[lo:hi]
        r = blk @ self.x - self.b[lo:hi]
        if self.extended:
            r += self.z[lo:hi]
        return self.torch.from_numpy(np.ascontiguousarray(blk.T @ r))

    def xupdate(self, scale, dx):
        self.x -= scale * dx.numpy()

    def err(self):
        return float(np.linalg.norm(self.x - self.xs))

    def state(self):
        return self.x.copy(), None if self.z is None else self.z.copy()

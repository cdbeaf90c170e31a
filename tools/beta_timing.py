"""Time beta_max resolution: device Lanczos (rebk_beta.cu)
against the host eigensolver (C2) and against torch's cuBLAS Gram +
cuSOLVER eigvalsh (C3, 16 GB built on the device).  Prints one line per
config: seconds, beta values and their relative difference.
usage: python tools/beta_timing.py [c2] [c3]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2001_04179_b200 as P  # noqa: E402
from paper_2001_04179_b200 import workloads  # noqa: E402


def c2():
    wl = workloads.build("c2")
    a, rp, cp = wl.problem.a, wl.row_partition, wl.col_partition
    a.device()  # upload outside the timed region
    P.device_beta_max(a, rp, cp)  # warm-up (module load, allocator)
    t0 = time.perf_counter()
    d = P.device_beta_max(a, rp, cp)
    td = time.perf_counter() - t0
    t0 = time.perf_counter()
    h = P.compute_beta_max(a, rp, cp)
    th = time.perf_counter() - t0
    dm = a.device()
    _, kr = dm.block_sigma1_sq(0, rp.pointers())
    _, kc = dm.block_sigma1_sq(1, cp.pointers())
    print(f"c2 device lanczos {td:.3f} s (steps rows {kr.min()}-{kr.max()}, cols {kc.min()}-{kc.max()}) | "
          f"host eigvalsh of block Grams {th:.3f} s ({os.cpu_count()} cores) | beta device {d[2]!r} host {h[2]!r} "
          f"rel diff {abs(d[2] - h[2]) / h[2]:.2e}")


def c3():
    import torch

    from paper_2001_04179_b200.matrix import DeviceMatrix

    t0 = time.perf_counter()
    wl = workloads.c3_device()
    tb = time.perf_counter() - t0
    m, n = wl.shape
    dm = DeviceMatrix.from_device_pointer(wl.a.data_ptr(), m, n, n, 0)
    dm.block_sigma1_sq(1, wl.col_ptr, max_steps=4)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sr, kr = dm.block_sigma1_sq(0, wl.row_ptr)
    sc, kc = dm.block_sigma1_sq(1, wl.col_ptr)
    td = time.perf_counter() - t0
    bd = max(float(np.max(sr / wl.row_w)), float(np.max(sc / wl.col_w)))
    # torch reference timing (cuBLAS Gram + cuSOLVER eigvalsh per block), as in workloads.c3_device
    a = wl.a
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bt = 0.0
    for lo, hi, wt in zip(wl.row_ptr[:-1], wl.row_ptr[1:], wl.row_w):
        blk = a[lo:hi]
        bt = max(bt, float(torch.linalg.eigvalsh(blk @ blk.T)[-1]) / wt)
    for lo, hi, wt in zip(wl.col_ptr[:-1], wl.col_ptr[1:], wl.col_w):
        blk = a[:, lo:hi]
        bt = max(bt, float(torch.linalg.eigvalsh(blk.T @ blk)[-1]) / wt)
    torch.cuda.synchronize()
    tt = time.perf_counter() - t0
    dm.close()
    print(f"c3 (build {tb:.1f} s) device lanczos {td:.3f} s (steps rows {kr.min()}-{kr.max()}, cols "
          f"{kc.min()}-{kc.max()}) | torch Gram+eigvalsh {tt:.3f} s | beta device {bd!r} torch {bt!r} "
          f"rel diff {abs(bd - bt) / bt:.2e}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["c2", "c3"]
    for w in which:
        {"c2": c2, "c3": c3}[w]()

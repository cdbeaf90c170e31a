"""C3 probe: 200000 x 10000 dense fp64 (16 GB) built on the device with torch,
run through librebk's device-pointer ABI.  Times a fixed number of
iterations (max_iters_only) and a solve to ||x - x*|| <= 1e-6 ||x*||.

Usage (GPU box): python tools/c3_probe.py [--m 200000] [--iters 50] [--solve]
"""
import argparse
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2001_04179_b200 import _lib  # noqa: E402
from paper_2001_04179_b200.matrix import DeviceMatrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=200000)
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--row-block", type=int, default=1000)
    ap.add_argument("--col-block", type=int, default=500)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--ab", default="", help="';'-separated env settings (A=1,B=2;...) timed one after the other")
    args = ap.parse_args()
    m, n = args.m, args.n
    dev = torch.device("cuda", 0)
    t0 = time.time()
    g = torch.Generator(device=dev).manual_seed(0)
    A = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
    xs = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    w = torch.randn(m, dtype=torch.float64, device=dev, generator=g)
    G = A.T @ A
    L = torch.linalg.cholesky(G)
    Ax = A @ xs
    r = w - A @ torch.cholesky_solve((A.T @ w)[:, None], L)[:, 0]
    r *= 0.1 * Ax.norm() / r.norm()
    b = Ax + r
    x_star = torch.cholesky_solve((A.T @ b)[:, None], L)[:, 0]
    del G, L, Ax, r, w
    torch.cuda.synchronize()
    print(f"[c3] instance built on device in {time.time() - t0:.1f} s", flush=True)

    dm = DeviceMatrix.from_device_pointer(A.data_ptr(), m, n, n, 0)
    row_ptr = np.array(list(range(0, m, args.row_block)) + [m], dtype=np.int64)
    col_ptr = np.array(list(range(0, n, args.col_block)) + [n], dtype=np.int64)
    wr = dm.block_frobenius_sq(0, row_ptr)
    wc = dm.block_frobenius_sq(1, col_ptr)
    # beta_max bound for alpha: power iteration on a few blocks is enough for a probe
    def beta(axis, ptr, wts, k=3):
        best = 0.0
        for bi in range(min(k, len(ptr) - 1)):
            blk = A[ptr[bi]:ptr[bi + 1], :] if axis == 0 else A[:, ptr[bi]:ptr[bi + 1]]
            s = torch.linalg.matrix_norm(blk, ord=2).item() ** 2 / wts[bi]
            best = max(best, s)
        return best
    bmax = max(beta(0, row_ptr, wr), beta(1, col_ptr, wc))
    alpha = 1.0 / bmax
    row_cum, col_cum = np.cumsum(wr), np.cumsum(wc)
    row_scale, col_scale = alpha / wr, alpha / wc
    print(f"[c3] beta_max(probe) = {bmax:.6g}, alpha = {alpha:.4g}", flush=True)

    def cfg(stop_mode, tol, max_iters):
        c = _lib.RebkCfg()
        c.algorithm = _lib.ALGO_CODES["rebk"]
        c.stop_mode = _lib.STOP_CODES[stop_mode]
        c.tol = tol
        c.check_stride = 1
        c.max_iters = max_iters
        k = _lib.philox_key(17)
        c.philox_key[0], c.philox_key[1] = int(k[0]), int(k[1])
        c.n_row_blocks = len(row_ptr) - 1
        c.row_ptr = _lib.i64ptr(row_ptr)
        c.row_cum = _lib.dptr(row_cum)
        c.row_total = float(row_cum[-1])
        c.row_scale = _lib.dptr(row_scale)
        c.n_col_blocks = len(col_ptr) - 1
        c.col_ptr = _lib.i64ptr(col_ptr)
        c.col_cum = _lib.dptr(col_cum)
        c.col_total = float(col_cum[-1])
        c.col_scale = _lib.dptr(col_scale)
        return c

    x = torch.zeros(n, dtype=torch.float64, device=dev)
    z = torch.empty(m, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    lib = _lib.load()

    def run(c):
        x.zero_()
        z.copy_(b)
        tr = _lib.RebkTrace()
        rc = lib.rebk_run_device(dm.handle, ctypes.byref(c), ctypes.c_void_p(b.data_ptr()),
                                 ctypes.c_void_p(x_star.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                 ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(stream.cuda_stream),
                                 ctypes.byref(tr))
        _lib.check(rc, "rebk_run_device")
        return tr

    alg = 8.0 * (m * args.col_block + args.row_block * n)
    c = cfg("max_iters_only", 1.0, args.iters)
    run(c)
    for _ in range(2):
        tr = run(c)
        us = 1e3 * tr.loop_ms / tr.iters
        print(f"[c3] {tr.iters} iterations: {tr.loop_ms:.2f} ms, {us:.1f} us/iter, "
              f"{alg / (us * 1e-6) / 1e9:.0f} GB/s algorithmic, grid {tr.grid_ctas}, path {tr.kernel_path}", flush=True)
    import os
    for setting in [v for v in args.ab.split(";") if v or args.ab]:
        kv = dict(e.split("=") for e in setting.split(",") if e)
        os.environ.update(kv)
        run(c)
        best = min(run(c).loop_ms for _ in range(3))
        print(f"[c3 ab] {setting or 'default':40s} {1e3 * best / args.iters:8.2f} us/iter", flush=True)
        for k in kv:
            del os.environ[k]
    if args.solve:
        tol = 1e-6 * x_star.norm().item()
        tr = run(cfg("oracle_error", tol, 5000))
        us = 1e3 * tr.loop_ms / max(tr.iters, 1)
        print(f"[c3] solve: ITER={tr.iters} converged={bool(tr.converged)} err={tr.final_error:.3e} "
              f"(tol {tol:.3e}) loop {tr.loop_ms:.1f} ms = {us:.1f} us/iter, "
              f"{alg / (us * 1e-6) / 1e9:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()

"""The row-sharded persistent kernel with the in-kernel cross-rank exchange
(rebk_shard_stream_kernel), with P ranks emulated in one
cooperative launch on one GPU (rebk_shard_run_virtual; B200_PROFILING.md:
ranks that wait on one another must run as ONE launch when there are fewer
GPUs than ranks).  The kernel code and the exchange protocol (inbox stores,
system-scope release flags, rank-order sums) are the ones a multi-GPU job
runs; only where the peer buffers live differs.

Gates: ITER equal to the reference's, x and z within 1e-10 of the
reference's iterates (golden vectors made by running the reference), x
bitwise identical on every rank, bitwise replay."""

import os

import numpy as np
import pytest

import paper_2001_04179_b200 as P
from paper_2001_04179_b200 import _lib

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RTOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def c1():
    from paper_2001_04179_b200.workloads import c1_matrix

    g = np.load(os.path.join(GOLD, "c1_golden.npz"))
    a = c1_matrix()
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=g["b"], x_star=g["x_star"], b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(2000, 100, "row"), P.contiguous_partition(500, 100, "col")
    cfg = P.SolverConfig(algorithm="rebk", alpha=float(g["alpha"]), seed=int(g["seed"]), max_iters=50_000,
                         row_partition=rp, col_partition=cp, stop=P.StoppingRule(tol=float(g["tol"])),
                         beta_max=float(g["beta"]))
    return g, a, prob, cfg


def device_cfg(prob, cfg, stop_mode="oracle_error", tol=None, max_iters=None, record=False, stride=1):
    ctx = P.prepare(prob, cfg)
    c = ctx.make_cfg(stop_mode=stop_mode, tol=cfg.stop.tol if tol is None else tol, stride=stride,
                     max_iters=cfg.max_iters if max_iters is None else max_iters, key=_lib.philox_key(cfg.seed),
                     record=record)
    return ctx, c


@pytest.mark.parametrize("vranks", [1, 2, 3, 4, 8])
def test_persistent_sharded_matches_reference_c1(vranks):
    from paper_2001_04179_b200.sharded import run_persistent_virtual

    g, a, prob, cfg = c1()
    ctx, c = device_cfg(prob, cfg)
    res = run_persistent_virtual(a, prob.b, g["x_star"], c, ctx._row_ptr, vranks)
    k = int(g["iters"])
    assert res["kernel_path"] == 9
    assert res["converged"] and res["iters"] == k, (res["iters"], k)
    assert rel(res["x"], g[f"x_{k}"]) <= RTOL
    assert rel(res["z"], g[f"z_{k}"]) <= RTOL
    for v in range(vranks):  # x is replicated bit for bit (rank-order sums everywhere)
        assert np.array_equal(res["x_all"][v], res["x"])
    res2 = run_persistent_virtual(a, prob.b, g["x_star"], c, ctx._row_ptr, vranks)
    assert np.array_equal(res2["x"], res["x"]) and np.array_equal(res2["z"], res["z"])


@pytest.mark.parametrize("vranks", [2, 4])
def test_persistent_sharded_snapshots_and_budget(vranks):
    """max_iters_only runs to the golden snapshot iterations (1, 10, 100):
    the exchange state carries correctly through the first iterations."""
    from paper_2001_04179_b200.sharded import run_persistent_virtual

    g, a, prob, cfg = c1()
    for k in (1, 10, 100):
        ctx, c = device_cfg(prob, cfg, stop_mode="max_iters_only", tol=1.0, max_iters=k)
        res = run_persistent_virtual(a, prob.b, g["x_star"], c, ctx._row_ptr, vranks)
        assert res["iters"] == k and not res["converged"]
        assert rel(res["x"], g[f"x_{k}"]) <= RTOL and rel(res["z"], g[f"z_{k}"]) <= RTOL


def test_persistent_sharded_ragged_blocks_fewer_rows_than_ranks():
    """Ragged partition (last row block of 3 rows < 8 ranks: some ranks own
    no rows of it) on a small problem against the oracle."""
    from oracle.rebk_oracle import OracleSolver
    from paper_2001_04179_b200.sharded import run_persistent_virtual

    g = np.random.default_rng(5)
    m, n = 403, 90
    a = g.standard_normal((m, n))
    xs = g.standard_normal(n)
    b = a @ xs + 0.05 * g.standard_normal(m)
    x_star = np.linalg.lstsq(a, b, rcond=None)[0]
    prob = P.ProblemInstance(a=P.Matrix.from_dense(a), b=b, x_star=x_star, b_perp=None,
                             meta=P.ProblemMeta(0, None, False, 0, 0.0))
    rp, cp = P.contiguous_partition(m, 50, "row"), P.contiguous_partition(n, 30, "col")
    tol = 1e-8 * float(np.linalg.norm(x_star))
    cfg = P.SolverConfig(algorithm="rebk", alpha=1.0, seed=7, max_iters=3000, row_partition=rp, col_partition=cp,
                         stop=P.StoppingRule(tol=tol), beta_max=0.3)
    ctx, c = device_cfg(prob, cfg)
    res = run_persistent_virtual(a, b, x_star, c, ctx._row_ptr, 8)
    orc = OracleSolver(a, b, rp.pointers(), cp.pointers(), 1.0, "rebk")
    ref = orc.run(7, 3000, tol, x_star)
    assert res["iters"] == ref["iters"] and res["converged"] == ref["converged"]
    assert rel(res["x"], ref["x"]) <= RTOL and rel(res["z"], ref["z"]) <= RTOL


@pytest.mark.slow
def test_persistent_sharded_c3_full_size_matches_single_gpu():
    """C3 at its BASELINE size (200000 x 10000, 16 GB) with 8 emulated ranks
    against the single-GPU streaming kernel on the same instance (itself
    pinned to the oracle in test_gpu_parity.py): same ITER, iterates within
    1e-10."""
    import ctypes

    import torch

    from paper_2001_04179_b200.matrix import DeviceMatrix
    from paper_2001_04179_b200.sharded import run_persistent_virtual
    from paper_2001_04179_b200.workloads import c3_device

    wl = c3_device()
    m, n = wl.shape
    tol = wl.rel_tol * float(wl.x_star.norm())
    c = wl.cfg("oracle_error", tol, 5000)
    dm = DeviceMatrix.from_device_pointer(wl.a.data_ptr(), m, n, n, 0)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    z = wl.b.clone()
    tr = _lib.RebkTrace()
    _lib.check(_lib.load().rebk_run_device(dm.handle, ctypes.byref(c), ctypes.c_void_p(wl.b.data_ptr()),
                                           ctypes.c_void_p(wl.x_star.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                           ctypes.c_void_p(z.data_ptr()), None, ctypes.byref(tr)), "run")
    dm.close()
    xs1, zs1 = x.cpu().numpy(), z.cpu().numpy()
    del x, z
    res = run_persistent_virtual(wl.a, wl.b, wl.x_star, c, wl.row_ptr, 8)
    assert res["iters"] == int(tr.iters) and res["converged"]
    assert rel(res["x"], xs1) <= RTOL and rel(res["z"], zs1) <= RTOL


def _ipc_rank_main(rank, world, port, out_dir):
    import os

    import numpy as np
    import torch.distributed as dist

    from paper_2001_04179_b200.sharded import ShardExchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # every process uses GPU 0: CUDA IPC maps a buffer of another PROCESS the
    # same way whether it lives on this GPU or on an NVLink peer
    x = ShardExchange(world, rank, 500, 10000, 0, dist.all_gather_object)
    ok, err = 1, ""
    try:
        for token in (1, 2, 7):
            x.probe(dist.barrier, token)
    except Exception as exc:  # reported through the file, the parent asserts
        ok, err = 0, repr(exc)
    np.savez(os.path.join(out_dir, f"ipc{rank}.npz"), ok=ok, err=err, grid=x.grid_ctas)
    dist.barrier()
    x.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_exchange_buffers_map_across_processes_over_cuda_ipc(world):
    """The multi-process setup of the in-kernel exchange on real CUDA: `world`
    processes (all on this one GPU) create their exchange buffers, export and
    map them over CUDA IPC (rebk_shard_xchg_ipc_handle / _open_peers) and
    probe the mappings with the protocol's own st.release.sys / ld.acquire.sys
    words, meeting at a host barrier in between (no kernel waits on another
    process's kernel, so this is legal on one GPU; the persistent kernels
    themselves are tested as emulated ranks in one launch above)."""
    import socket
    import tempfile

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_ipc_rank_main, args=(world, port, d), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"ipc{r}.npz")) for r in range(world)]
    for r, o in enumerate(outs):
        assert int(o["ok"]) == 1, (r, str(o["err"]))
        assert int(o["grid"]) == int(outs[0]["grid"])

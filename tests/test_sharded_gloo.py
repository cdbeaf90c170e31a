"""Row-sharded REBK (config 3's multi-GPU layout) across 2 CPU ranks over
gloo: the sharded loop (paper_2001_04179_b200.sharded.run_sharded) with the
CPU restatement of the per-rank kernels must reproduce the single-process
oracle (same block sequence): ITER equal, x and z within 1e-12."""

import os
import socket
import tempfile

import numpy as np
import pytest

from oracle.rebk_oracle import OracleRng, OracleSolver


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def problem():
    g = np.random.default_rng(3)
    a = g.standard_normal((83, 31))
    xs = g.standard_normal(31)
    b = a @ xs + 0.05 * g.standard_normal(83)
    x_star = np.linalg.lstsq(a, b, rcond=None)[0]
    row_ptr = np.r_[np.arange(0, 83, 7), 83]
    col_ptr = np.r_[np.arange(0, 31, 6), 31]
    return a, b, x_star, row_ptr, col_ptr


def reference_run(max_iters, tol):
    a, b, x_star, row_ptr, col_ptr = problem()
    orc = OracleSolver(a, b, row_ptr, col_ptr, 1.1, "rebk")
    return orc, orc.run(11, max_iters, tol, x_star)


def _rank_main(rank, world, port, out_dir, max_iters, tol):
    import torch
    import torch.distributed as dist

    from oracle.shard_oracle import NumpyShardBackend
    from paper_2001_04179_b200.sharded import ShardPlan, owned_rows, run_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b, x_star, row_ptr, col_ptr = problem()
    orc = OracleSolver(a, b, row_ptr, col_ptr, 1.1, "rebk")
    picks = orc.picks(OracleRng(11), max_iters)
    plan = ShardPlan(row_ptr, col_ptr, np.asarray(orc.row_scales), np.asarray(orc.col_scales), picks)
    rows, ranges = owned_rows(row_ptr, world, rank)
    be = NumpyShardBackend(a[rows], b[rows], x_star, True)
    res = run_sharded(be, plan, ranges, max_iters, tol, allreduce=lambda t: dist.all_reduce(t))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), rows=rows, x=res["x"], z=res["z_local"], iters=res["iters"],
             conv=res["converged"], err=res["final_error"])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_loop_matches_single_process_oracle(world):
    import torch.multiprocessing as mp

    max_iters, tol = 4000, 1e-9
    _, ref = reference_run(max_iters, tol)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(world, free_port(), d, max_iters, tol), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    z = np.zeros(83)
    for o in outs:
        assert int(o["iters"]) == ref["iters"] and bool(o["conv"]) == ref["converged"]
        assert np.linalg.norm(o["x"] - ref["x"]) <= 1e-12 * np.linalg.norm(ref["x"])
        z[o["rows"]] = o["z"]
    assert np.linalg.norm(z - ref["z"]) <= 1e-12 * np.linalg.norm(ref["z"])
    # x is replicated bit for bit (every rank applies the same reduced dx)
    for o in outs[1:]:
        assert np.array_equal(o["x"], outs[0]["x"])


def test_row_ownership_partitions_every_block():
    from paper_2001_04179_b200.sharded import owned_rows

    row_ptr = np.array([0, 100, 200, 280, 281])
    for world in (1, 2, 3, 8):
        seen = np.zeros(281, dtype=int)
        for r in range(world):
            rows, ranges = owned_rows(row_ptr, world, r)
            seen[rows] += 1
            assert ranges[-1, 1] == rows.size
            for bi in range(4):
                blk = rows[ranges[bi, 0]:ranges[bi, 1]]
                assert np.all((blk >= row_ptr[bi]) & (blk < row_ptr[bi + 1]))
        assert np.all(seen == 1)


class _FakeXchgLib:
    """Records the C-ABI calls ShardExchange makes (no GPU on this host): the
    per-rank CTA count it reports, the IPC handle it exports, and the handle
    table it is asked to open."""

    def __init__(self, rank, ctas):
        self.rank, self.ctas = rank, ctas
        self.created = None
        self.opened = None

    def rebk_shard_grid_ctas(self, device, out):
        out._obj.value = self.ctas
        return 0

    def rebk_shard_xchg_create(self, P, rank, nJ, n, G, device, out):
        self.created = (P, rank, nJ, n, G, device)
        out._obj.value = 1000 + rank
        return 0

    def rebk_shard_xchg_ipc_handle(self, h, buf):
        buf.raw = bytes([self.rank]) * 64
        return 0

    def rebk_shard_xchg_open_peers(self, h, handles):
        self.opened = bytes(handles)
        return 0

    def rebk_shard_xchg_destroy(self, h):
        return 0


def _xchg_rank_main(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2001_04179_b200.sharded import ShardExchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = _FakeXchgLib(rank, ctas=148 - 3 * rank)  # ranks report different CTA counts
    x = ShardExchange(world, rank, 500, 10000, rank, dist.all_gather_object, lib=lib)
    np.savez(os.path.join(out_dir, f"x{rank}.npz"), created=np.asarray(lib.created),
             opened=np.frombuffer(lib.opened, dtype=np.uint8), grid=x.grid_ctas)
    x.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_exchange_setup_agrees_across_ranks(world):
    """The multi-GPU setup of the in-kernel exchange (sharded.ShardExchange)
    over gloo: every rank agrees on the minimum CTA count (the dx exchange
    pairs CTA g with CTA g, so the x split must match), creates its buffer
    with its own rank, and receives every rank's IPC handle in rank order."""
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_xchg_rank_main, args=(world, free_port(), d), nprocs=world, join=True)
        outs = [np.load(os.path.join(d, f"x{r}.npz")) for r in range(world)]
    want_g = 148 - 3 * (world - 1)
    want_handles = b"".join(bytes([r]) * 64 for r in range(world))
    for r, o in enumerate(outs):
        assert int(o["grid"]) == want_g
        assert o["created"].tolist() == [world, r, 500, 10000, want_g, r]
        assert o["opened"].tobytes() == want_handles

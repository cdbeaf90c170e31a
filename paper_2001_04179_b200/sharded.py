"""Row-sharded REBK over P ranks (BASELINE config 3).

Layout: every row block I_b is split across all ranks — local row q of
I_b lives on rank floor(q * P / |I_b|) — so the row step is balanced and no
rank ever needs another rank's rows.  z and b follow the rows; x is
replicated.  One iteration (step_rebk, solvers.py:324-337):

    u_p  = A_p[:, J]ᵀ z_p          -> allreduce(u)   (|J| doubles)
    z_p -= s_J A_p[:, J] u
    dx_p = A_p[I_p, :]ᵀ (A_p[I_p, :] x - b_p + z_p)
                                   -> allreduce(dx)  (n doubles)
    x   -= s_I dx

The stop check needs no communication (x is replicated, every rank computes
the same ||x - x*||).  The block sequence is shared: every rank expands the
same Philox stream.

The per-rank arithmetic is a backend: :class:`CudaShardBackend` (librebk's
``rebk_shard_*`` kernels, device buffers, allreduce over NCCL via
torch.distributed).  Tests drive the same loop with a CPU restatement under
gloo (oracle/shard_oracle.py) to check the sharding logic.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib


def owned_rows(row_ptr: np.ndarray, nranks: int, rank: int) -> tuple[np.ndarray, np.ndarray]:
    """Global rows owned by `rank` (sorted) and, per row block, the [lo, hi)
    range of those rows in the rank's local ordering."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    rows, ranges = [], np.zeros((row_ptr.size - 1, 2), dtype=np.int64)
    pos = 0
    for b in range(row_ptr.size - 1):
        lo, nb = int(row_ptr[b]), int(row_ptr[b + 1] - row_ptr[b])
        q0 = -(-rank * nb // nranks)          # ceil(rank * nb / P)
        q1 = -(-(rank + 1) * nb // nranks)
        rows.append(np.arange(lo + q0, lo + q1, dtype=np.int64))
        ranges[b] = (pos, pos + (q1 - q0))
        pos += q1 - q0
    return np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64), ranges


@dataclass
class ShardPlan:
    """Everything every rank shares: partitions, scales, the pick sequence."""

    row_ptr: np.ndarray
    col_ptr: np.ndarray | None
    row_scale: np.ndarray
    col_scale: np.ndarray | None
    picks: np.ndarray  # (max_iters, 2): column block (or -1), row block


def plan_from_context(ctx, max_iters: int) -> ShardPlan:
    """Shared plan from a SolverContext built on the full matrix (the
    reference's sampler arrays), with the pick sequence expanded on the
    device from the run's Philox stream."""
    cfg = ctx.make_cfg(stop_mode="max_iters_only", tol=1.0, stride=1, max_iters=max_iters,
                       key=_lib.philox_key(ctx.config.seed))
    picks = np.empty((max_iters, 2), dtype=np.int32)
    if max_iters:
        rc = _lib.load().rebk_sample_sequence(ctypes.byref(cfg), 1, max_iters,
                                              picks.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        _lib.check(rc, "rebk_sample_sequence")
    return ShardPlan(ctx._row_ptr, ctx._col_ptr if ctx.extended else None, ctx._row_scale,
                     ctx._col_scale if ctx.extended else None, picks)


class CudaShardBackend:
    """This rank's rows of A on its GPU; all state in device memory."""

    def __init__(self, a_local: np.ndarray, b_local: np.ndarray, x_star: np.ndarray | None, extended: bool,
                 device: int = 0):
        import torch

        from .matrix import DeviceMatrix

        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.lib = _lib.load()
        self.m_local, self.n = a_local.shape
        self.extended = extended
        # an empty shard still needs a valid matrix: keep one zero row
        a = a_local if self.m_local else np.zeros((1, self.n))
        self.dm = DeviceMatrix(a, device)
        t = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(self.dev)
        self.b = t(b_local if self.m_local else np.zeros(1))
        self.z = self.b.clone() if extended else None
        self.x = torch.zeros(self.n, dtype=torch.float64, device=self.dev)
        self.xs = None if x_star is None else t(x_star)
        self.dx = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        self.err_buf = torch.empty(1, dtype=torch.float64, device=self.dev)
        self.rows_cache: dict = {}

    @classmethod
    def from_device(cls, a_local, b_local, x_star, extended: bool, device: int = 0) -> "CudaShardBackend":
        """Shard already on the GPU (torch CUDA tensors, e.g. gathered from a
        device-built instance): no host round trip of A."""
        import torch

        from .matrix import DeviceMatrix

        self = cls.__new__(cls)
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.lib = _lib.load()
        self.m_local, self.n = int(a_local.shape[0]), int(a_local.shape[1])
        self.extended = extended
        a = a_local.contiguous() if self.m_local else torch.zeros((1, self.n), dtype=torch.float64, device=self.dev)
        self._a_keep = a
        self.dm = DeviceMatrix.from_device_pointer(a.data_ptr(), a.shape[0], self.n, self.n, device)
        self.b = (b_local if self.m_local else torch.zeros(1, dtype=torch.float64, device=self.dev)).clone()
        self.z = self.b.clone() if extended else None
        self.x = torch.zeros(self.n, dtype=torch.float64, device=self.dev)
        self.xs = None if x_star is None else x_star.clone()
        self.dx = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        self.err_buf = torch.empty(1, dtype=torch.float64, device=self.dev)
        self.rows_cache = {}
        return self

    def err2_into(self, out):
        """||x - x*||^2 into the device scalar `out` (no host sync)."""
        _lib.check(self.lib.rebk_shard_err2(self.n, ctypes.c_void_p(self.x.data_ptr()),
                                            ctypes.c_void_p(self.xs.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                            self._stream()), "err2")

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.dev).cuda_stream)

    def colstep(self, c_lo: int, c_hi: int):
        u = self.torch.empty(c_hi - c_lo, dtype=self.torch.float64, device=self.dev)
        if self.m_local:
            _lib.check(self.lib.rebk_shard_colstep(self.dm.handle, c_lo, c_hi, ctypes.c_void_p(self.z.data_ptr()),
                                                   ctypes.c_void_p(u.data_ptr()), self._stream()), "colstep")
        else:
            u.zero_()
        return u

    def zupdate(self, c_lo: int, c_hi: int, scale: float, u):
        if self.m_local:
            _lib.check(self.lib.rebk_shard_zupdate(self.dm.handle, c_lo, c_hi, scale, ctypes.c_void_p(u.data_ptr()),
                                                   ctypes.c_void_p(self.z.data_ptr()), self._stream()), "zupdate")

    def rowstep(self, lo: int, hi: int):
        key = (lo, hi)
        rows = self.rows_cache.get(key)
        if rows is None:
            rows = self.torch.arange(lo, hi, dtype=self.torch.int64, device=self.dev)
            self.rows_cache[key] = rows
        zp = ctypes.c_void_p(self.z.data_ptr()) if self.extended else None
        _lib.check(self.lib.rebk_shard_rowstep(self.dm.handle, ctypes.c_void_p(rows.data_ptr()), hi - lo,
                                               ctypes.c_void_p(self.x.data_ptr()), ctypes.c_void_p(self.b.data_ptr()),
                                               zp, ctypes.c_void_p(self.dx.data_ptr()), self._stream()), "rowstep")
        return self.dx

    def xupdate(self, scale: float, dx):
        _lib.check(self.lib.rebk_shard_xupdate(self.n, scale, ctypes.c_void_p(dx.data_ptr()),
                                               ctypes.c_void_p(self.x.data_ptr()), self._stream()), "xupdate")

    def err(self) -> float:
        _lib.check(self.lib.rebk_shard_err2(self.n, ctypes.c_void_p(self.x.data_ptr()),
                                            ctypes.c_void_p(self.xs.data_ptr()), ctypes.c_void_p(self.err_buf.data_ptr()),
                                            self._stream()), "err2")
        return float(np.sqrt(self.err_buf.item()))

    def state(self):
        z = None if self.z is None else self.z.cpu().numpy()[: self.m_local]
        return self.x.cpu().numpy(), z


def run_sharded(backend, plan: ShardPlan, ranges: np.ndarray, max_iters: int, tol: float, stride: int = 1,
                mode: str = "oracle_error", allreduce=None) -> dict:
    """The run() loop (solvers.py:425-474) on one rank; `allreduce(t)` sums a
    vector over all ranks in place (identity for a single rank)."""
    allreduce = allreduce or (lambda t: None)
    checking = mode == "oracle_error"
    final, converged, iters = None, False, 0
    if checking:
        final = backend.err()
        converged = final <= tol
    if not converged:
        for k in range(1, max_iters + 1):
            j, i = int(plan.picks[k - 1, 0]), int(plan.picks[k - 1, 1])
            if backend.extended:
                c_lo, c_hi = int(plan.col_ptr[j]), int(plan.col_ptr[j + 1])
                u = backend.colstep(c_lo, c_hi)
                allreduce(u)
                backend.zupdate(c_lo, c_hi, float(plan.col_scale[j]), u)
            lo, hi = int(ranges[i, 0]), int(ranges[i, 1])
            dx = backend.rowstep(lo, hi)
            allreduce(dx)
            backend.xupdate(float(plan.row_scale[i]), dx)
            if checking and k % stride == 0:
                final = backend.err()
                if final <= tol:
                    converged, iters = True, k
                    break
        else:
            iters = max_iters
            if checking and max_iters % stride != 0:
                final = backend.err()
                converged = final <= tol
    x, z = backend.state()
    return dict(iters=iters, converged=converged, final_error=final, x=x, z_local=z)


def run_sharded_chunked(backend, plan: ShardPlan, ranges: np.ndarray, max_iters: int, tol: float,
                        stride: int = 1, allreduce=None, chunk: int = 32) -> dict:
    """run_sharded without a host synchronisation per check: the errors of a
    chunk of iterations are written on the device and read once per chunk.
    x and z are snapshotted at the chunk start; when a check inside the chunk
    crosses tol, the chunk is replayed from the snapshot up to exactly that
    iteration (the kernels and the fixed-size allreduces are deterministic),
    so the returned state is the reference's (solvers.py:444-474)."""
    import torch

    allreduce = allreduce or (lambda t: None)
    errs = torch.empty(chunk, dtype=torch.float64, device=backend.dev)

    def iterate(k):
        j, i = int(plan.picks[k - 1, 0]), int(plan.picks[k - 1, 1])
        if backend.extended:
            c_lo, c_hi = int(plan.col_ptr[j]), int(plan.col_ptr[j + 1])
            u = backend.colstep(c_lo, c_hi)
            allreduce(u)
            backend.zupdate(c_lo, c_hi, float(plan.col_scale[j]), u)
        lo, hi = int(ranges[i, 0]), int(ranges[i, 1])
        dx = backend.rowstep(lo, hi)
        allreduce(dx)
        backend.xupdate(float(plan.row_scale[i]), dx)

    final = backend.err()
    converged, iters = final <= tol, 0
    k = 0
    while not converged and k < max_iters:
        cnt = min(chunk, max_iters - k)
        x0 = backend.x.clone()
        z0 = backend.z.clone() if backend.extended else None
        checks = []
        for t in range(cnt):
            iterate(k + t + 1)
            if (k + t + 1) % stride == 0:
                backend.err2_into(errs[t:t + 1])
                checks.append(t)
        hit = None
        if checks:
            vals = errs[:cnt].cpu().numpy()
            e = np.full(cnt, np.inf)
            e[checks] = np.sqrt(vals[checks])  # only the checked slots were written
            for t in checks:
                if e[t] <= tol:
                    hit = t
                    break
        if hit is not None:
            if hit + 1 < cnt:  # replay to the crossing iteration exactly
                backend.x.copy_(x0)
                if z0 is not None:
                    backend.z.copy_(z0)
                for t in range(hit + 1):
                    iterate(k + t + 1)
            converged, iters, final = True, k + hit + 1, float(e[hit])
            break
        if checks:
            final = float(e[checks[-1]])
        k += cnt
    if not converged:
        iters = max_iters
        if max_iters % stride != 0:
            final = backend.err()
            converged = final <= tol
    x, z = backend.state()
    return dict(iters=iters, converged=converged, final_error=final, x=x, z_local=z)


def run_virtual_ranks(backends: list, plan: ShardPlan, ranges: list, max_iters: int, tol: float,
                      stride: int = 1) -> dict:
    """The sharded iteration for several ranks driven in lockstep by one
    process (one GPU can host them; the "allreduce" is a sum of the ranks'
    device vectors in rank order).  Used to exercise the multi-rank kernels
    where only one GPU is available."""
    first = backends[0]
    checking = True
    final = first.err()
    converged, iters = final <= tol, 0
    if not converged:
        for k in range(1, max_iters + 1):
            j, i = int(plan.picks[k - 1, 0]), int(plan.picks[k - 1, 1])
            if first.extended:
                c_lo, c_hi = int(plan.col_ptr[j]), int(plan.col_ptr[j + 1])
                us = [be.colstep(c_lo, c_hi) for be in backends]
                u = us[0].clone()
                for v in us[1:]:
                    u += v
                for be in backends:
                    be.zupdate(c_lo, c_hi, float(plan.col_scale[j]), u)
            dxs = [be.rowstep(int(r[i, 0]), int(r[i, 1])).clone() for be, r in zip(backends, ranges)]
            dx = dxs[0]
            for v in dxs[1:]:
                dx += v
            for be in backends:
                be.xupdate(float(plan.row_scale[i]), dx)
            if checking and k % stride == 0:
                final = first.err()
                if final <= tol:
                    converged, iters = True, k
                    break
        else:
            iters = max_iters
    return dict(iters=iters, converged=converged, final_error=final,
                states=[be.state() for be in backends])


# ---------------------------------------------------------------- native (C++) driver
def nccl_library_path() -> str:
    """The libnccl.so.2 torch loads (the nvidia-nccl wheel), else the loader default."""
    try:
        import nvidia.nccl

        import os

        for base in nvidia.nccl.__path__:
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except Exception:
        pass
    return "libnccl.so.2"


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _lib.check(_lib.load().rebk_nccl_get_unique_id(nccl_library_path().encode(), buf), "rebk_nccl_get_unique_id")
    return buf.raw


class NcclComm:
    """NCCL communicator owned by librebk (rebk_nccl_comm_create); every rank
    passes the same 128-byte unique id (rank 0's, distributed by the caller)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int = 0):
        h = ctypes.c_void_p()
        _lib.check(_lib.load().rebk_nccl_comm_create(nccl_library_path().encode(), uid, nranks, rank, device,
                                                     ctypes.byref(h)), "rebk_nccl_comm_create")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().rebk_nccl_comm_destroy(self.handle)
            self.handle = None


def run_sharded_native(backend: CudaShardBackend, comm: NcclComm, plan: ShardPlan, ranges: np.ndarray,
                       max_iters: int, tol: float, stride: int = 1, chunk: int = 32) -> dict:
    """run_sharded_chunked with the whole loop in C++ (rebk_shard_run): the
    per-rank kernels and both NCCL allreduces of every iteration are issued
    from librebk on one stream, no Python per iteration."""
    import torch

    args = _lib.RebkShardRunArgs()
    picks = np.ascontiguousarray(plan.picks[:max_iters], dtype=np.int32)
    row_ptr = np.ascontiguousarray(plan.row_ptr, dtype=np.int64)
    row_scale = np.ascontiguousarray(plan.row_scale, dtype=np.float64)
    rng = np.ascontiguousarray(ranges, dtype=np.int64)
    keep = [picks, row_ptr, row_scale, rng]
    args.max_iters, args.stride, args.tol, args.chunk = int(max_iters), int(stride), float(tol), int(chunk)
    args.extended = 1 if backend.extended else 0
    args.picks = picks.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    args.n_picks = picks.shape[0]
    if backend.extended:
        col_ptr = np.ascontiguousarray(plan.col_ptr, dtype=np.int64)
        col_scale = np.ascontiguousarray(plan.col_scale, dtype=np.float64)
        keep += [col_ptr, col_scale]
        args.n_col_blocks = col_ptr.size - 1
        args.col_ptr, args.col_scale = _lib.i64ptr(col_ptr), _lib.dptr(col_scale)
    args.n_row_blocks = row_ptr.size - 1
    args.row_ptr, args.row_scale = _lib.i64ptr(row_ptr), _lib.dptr(row_scale)
    args.local_ranges = _lib.i64ptr(rng)
    rows = torch.arange(max(backend.m_local, 1), dtype=torch.int64, device=backend.dev)
    args.local_rows_dev = rows.data_ptr()
    args.b_dev, args.x_dev = backend.b.data_ptr(), backend.x.data_ptr()
    args.z_dev = backend.z.data_ptr() if backend.extended else None
    args.xs_dev = backend.xs.data_ptr()
    torch.cuda.synchronize(backend.dev)  # x, z, b initialised on torch's stream
    it = ctypes.c_int64()
    conv = ctypes.c_int32()
    err = ctypes.c_double()
    _lib.check(_lib.load().rebk_shard_run(backend.dm.handle, comm.handle, ctypes.byref(args), ctypes.byref(it),
                                          ctypes.byref(conv), ctypes.byref(err)), "rebk_shard_run")
    del keep
    x, z = backend.state()
    return dict(iters=int(it.value), converged=bool(conv.value), final_error=float(err.value), x=x, z_local=z)


# ---------------------------------------------------------------- persistent kernel with the in-kernel exchange
def shard_layout(row_ptr: np.ndarray, nranks: int) -> tuple[list[np.ndarray], np.ndarray]:
    """Every rank's global rows and its local row ranges per row block
    ([nranks][n_row_blocks][2]), the interleaving of owned_rows."""
    rows, ranges = zip(*(owned_rows(row_ptr, nranks, r) for r in range(nranks)))
    return list(rows), np.ascontiguousarray(np.stack(ranges), dtype=np.int64)


def _as_device(t, dev):
    import torch

    if isinstance(t, torch.Tensor):
        return t.to(dev, dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(t, dtype=np.float64)).to(dev)


def run_persistent_virtual(a, b, x_star, cfg, row_ptr: np.ndarray, vranks: int, x0=None, z0=None,
                           device: int = 0) -> dict:
    """The row-sharded persistent kernel (rebk_shard_stream_kernel) with
    `vranks` ranks emulated in one cooperative launch on one GPU
    (rebk_shard_run_virtual): each emulated rank gets its interleaved rows
    of every row block, its own x copy and its own exchange buffer, and the
    ranks exchange u and dx partials through those buffers exactly as real
    ranks do through peer memory.  `cfg` is the single-GPU rebk_cfg (global
    partitions and sampler arrays).  Returns x (rank 0's copy), every rank's
    x (bitwise replicated), z in global row order and the trace."""
    import torch

    from .matrix import DeviceMatrix

    dev = torch.device("cuda", device)
    a_d, b_d = _as_device(a, dev), _as_device(b, dev)
    m, n = int(a_d.shape[0]), int(a_d.shape[1])
    rows, ranges = shard_layout(row_ptr, vranks)
    perm = torch.from_numpy(np.concatenate(rows)).to(dev)
    a_st = a_d.index_select(0, perm).contiguous()
    b_st = b_d.index_select(0, perm).contiguous()
    z_st = (b_d if z0 is None else _as_device(z0, dev)).index_select(0, perm).contiguous()
    x_all = (torch.zeros(n, dtype=torch.float64, device=dev) if x0 is None else _as_device(x0, dev)).repeat(vranks, 1)
    xs_d = None if x_star is None else _as_device(x_star, dev)
    rows_per = np.asarray([r.size for r in rows], dtype=np.int64)
    dm = DeviceMatrix.from_device_pointer(a_st.data_ptr(), m, n, n, device)
    tr = _lib.RebkTrace()
    errs = None
    if cfg.record_errors:
        errs = np.zeros(max(1, cfg.max_iters // max(1, cfg.check_stride) + 2))
        tr.errors, tr.errors_cap = _lib.dptr(errs), errs.size
    torch.cuda.synchronize(dev)
    try:
        _lib.check(_lib.load().rebk_shard_run_virtual(
            dm.handle, int(vranks), _lib.i64ptr(rows_per), _lib.i64ptr(ranges), ctypes.byref(cfg),
            ctypes.c_void_p(b_st.data_ptr()), ctypes.c_void_p(0 if xs_d is None else xs_d.data_ptr()),
            ctypes.c_void_p(x_all.data_ptr()), ctypes.c_void_p(z_st.data_ptr()),
            ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream), ctypes.byref(tr)), "rebk_shard_run_virtual")
    finally:
        dm.close()
    z = torch.empty_like(z_st)
    z[perm] = z_st
    xs_all = x_all.cpu().numpy()
    return dict(iters=int(tr.iters), converged=bool(tr.converged), final_error=float(tr.final_error),
                x=xs_all[0], x_all=xs_all, z=z.cpu().numpy(), loop_ms=float(tr.loop_ms), grid_ctas=int(tr.grid_ctas),
                kernel_path=int(tr.kernel_path), errors=errs, n_checks=int(tr.n_checks))


def exchange_ipc_handles(handle: bytes, all_gather_object) -> bytes:
    """Every rank's 64-byte CUDA IPC handle, concatenated in rank order
    (`all_gather_object(list, obj)` is torch.distributed's, or a stand-in)."""
    got = [None] * _world_size(all_gather_object)
    all_gather_object(got, bytes(handle))
    if any(h is None or len(h) != 64 for h in got):
        raise RuntimeError("IPC handle exchange returned a malformed handle")
    return b"".join(got)


def _world_size(all_gather_object):
    ws = getattr(all_gather_object, "world_size", None)
    if ws is not None:
        return int(ws)
    import torch.distributed as dist

    return dist.get_world_size()


class ShardExchange:
    """This rank's exchange buffer for rebk_shard_run_device, with every
    peer's buffer mapped over CUDA IPC (one process per GPU, one node).

    Collective: every rank constructs it with the same nJ_cap / n; the CTAs
    per rank are agreed as the minimum over ranks (all ranks must split x
    identically for the CTA-to-CTA dx exchange)."""

    def __init__(self, nranks: int, rank: int, nJ_cap: int, n: int, device: int, all_gather_object,
                 lib=None):
        self.lib = lib or _lib.load()
        g = ctypes.c_int()
        _lib.check(self.lib.rebk_shard_grid_ctas(device, ctypes.byref(g)), "rebk_shard_grid_ctas")
        gs = [None] * nranks
        all_gather_object(gs, int(g.value))
        self.grid_ctas = int(min(gs))
        h = ctypes.c_void_p()
        _lib.check(self.lib.rebk_shard_xchg_create(nranks, rank, int(nJ_cap), int(n), self.grid_ctas, device,
                                                   ctypes.byref(h)), "rebk_shard_xchg_create")
        self.handle = h
        buf = ctypes.create_string_buffer(64)
        _lib.check(self.lib.rebk_shard_xchg_ipc_handle(h, buf), "rebk_shard_xchg_ipc_handle")
        allh = exchange_ipc_handles(buf.raw, all_gather_object)
        _lib.check(self.lib.rebk_shard_xchg_open_peers(h, allh), "rebk_shard_xchg_open_peers")
        self.nranks, self.rank, self.device = nranks, rank, device

    def run(self, dm, cfg, ranges: np.ndarray, b_dev, xs_dev, x_dev, z_dev, stream) -> "_lib.RebkTrace":
        """One solve of this rank's shard (all device buffers; see rebk.h)."""
        rng = np.ascontiguousarray(ranges, dtype=np.int64)
        tr = _lib.RebkTrace()
        _lib.check(self.lib.rebk_shard_run_device(
            dm.handle, self.handle, ctypes.byref(cfg), _lib.i64ptr(rng), ctypes.c_void_p(b_dev),
            ctypes.c_void_p(xs_dev or 0), ctypes.c_void_p(x_dev), ctypes.c_void_p(z_dev or 0), ctypes.c_void_p(stream),
            ctypes.byref(tr)), "rebk_shard_run_device")
        return tr

    def probe(self, barrier, token: int = 1) -> None:
        """Collective check of the peer mappings before any persistent kernel
        depends on them: every rank stores a token word into every rank's
        buffer with the protocol's own st.release.sys, the ranks meet at
        `barrier()` (host side), then each rank verifies that all words
        arrived.  Raises RuntimeError naming the count of missing ranks."""
        _lib.check(self.lib.rebk_shard_xchg_probe(self.handle, 0, int(token), None), "rebk_shard_xchg_probe")
        barrier()
        missing = ctypes.c_int(-1)
        _lib.check(self.lib.rebk_shard_xchg_probe(self.handle, 1, int(token), ctypes.byref(missing)),
                   "rebk_shard_xchg_probe")
        barrier()
        if missing.value != 0:
            raise RuntimeError(f"rank {self.rank}: the probe words of {missing.value} of {self.nranks} ranks did not "
                               "arrive through the peer mapping")

    def close(self):
        if getattr(self, "handle", None):
            self.lib.rebk_shard_xchg_destroy(self.handle)
            self.handle = None

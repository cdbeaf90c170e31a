"""CPU restatement of the reference's REBK path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference code it restates (paths relative to
/root/reference/pkg/src/kaczmarz/).  The random stream lives in a
third-party dependency absent from /root/reference: numpy (effective pin
2.3.x; the reference's pyproject.toml:10-13 pins only numpy>=1.24).  Its
published algorithms are restated here in pure Python integers:
  * SeedSequence (O'Neill seed_seq hashing, pool size 4) — numpy
    bit_generator.pyx, used by Rng.__init__ (sampling.py:33-37);
  * Philox4x64-10 (Salmon et al., SC'11) with numpy's counter discipline
    (counter incremented before each 4-word block) — used by Rng.uniform
    (sampling.py:43-45) as (u64 >> 11) * 2^-53.
The linear algebra uses the same numpy operations, in the same order, as
the reference, so on the same machine the oracle reproduces the reference
bit for bit (checked against the golden vectors).
"""

from __future__ import annotations

import time

import numpy as np

MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF


# -- numpy SeedSequence (restated) ---------------------------------------------

def _words(v: int) -> list[int]:
    v = int(v)
    if v < 0:
        raise ValueError("negative entropy")
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & MASK32)
        v >>= 32
    return out


def seedseq_state_u64(seed: int, spawn_key=(), n_words64: int = 2) -> list[int]:
    """SeedSequence(seed, spawn_key).generate_state(n, uint64)."""
    INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
    INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
    MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
    run = _words(seed)
    spawn = [w for k in spawn_key for w in _words(k)]
    if spawn and len(run) < 4:
        run = run + [0] * (4 - len(run))
    ent = run + spawn
    hc = [INIT_A]

    def hashmix(v):
        v ^= hc[0]
        hc[0] = (hc[0] * MULT_A) & MASK32
        v = (v * hc[0]) & MASK32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & MASK32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    hb = INIT_B
    st = []
    for i in range(2 * n_words64):
        v = pool[i % 4] ^ hb
        hb = (hb * MULT_B) & MASK32
        v = (v * hb) & MASK32
        st.append(v ^ (v >> 16))
    return [st[2 * i] | (st[2 * i + 1] << 32) for i in range(n_words64)]


# -- Philox4x64-10 (restated) --------------------------------------------------

def philox4x64_10(ctr: list[int], key: list[int]) -> list[int]:
    M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
    W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
    c = list(ctr)
    k0, k1 = key
    for rnd in range(10):
        if rnd:
            k0 = (k0 + W0) & MASK64
            k1 = (k1 + W1) & MASK64
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> 64, p0 & MASK64
        hi1, lo1 = p1 >> 64, p1 & MASK64
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


class OracleRng:
    """Rng(seed) restated: draw d is word d%4 of Philox(counter=d//4+1, key)."""

    def __init__(self, seed: int, spawn_key=()):
        self.key = seedseq_state_u64(seed, spawn_key)
        self.draws = 0
        self._blk = -1
        self._buf = None

    def word(self, d: int) -> int:
        blk = d >> 2
        if blk != self._blk:
            c = blk + 1
            self._buf = philox4x64_10([c & MASK64, c >> 64, 0, 0], self.key)
            self._blk = blk
        return self._buf[d & 3]

    def uniform(self) -> float:
        w = self.word(self.draws)
        self.draws += 1
        return float(w >> 11) * (1.0 / 9007199254740992.0)


class NumpyRng:
    """The same stream through numpy's C Philox (the reference's own
    generator) — used only to time the CPU reference arm at full speed."""

    def __init__(self, seed: int):
        self._g = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))

    def uniform(self) -> float:
        return float(self._g.random())


# -- sampler (sampling.py:119-145, matrix.py:170-189) ---------------------------

def _sel(blk):
    """Contiguous blocks slice (views, as the reference does for ranges);
    index sets copy (matrix.py:153-168, solvers.py:115-120)."""
    if isinstance(blk, range):
        return slice(blk.start, blk.stop)
    arr = np.asarray(blk, dtype=np.int64)
    if arr.size > 1 and np.all(np.diff(arr) == 1):
        return slice(int(arr[0]), int(arr[-1]) + 1)
    if arr.size == 1:
        return slice(int(arr[0]), int(arr[0]) + 1)
    return arr


def blocks_from_ptr(ptr) -> list:
    ptr = np.asarray(ptr, dtype=np.int64)
    return [range(int(lo), int(hi)) for lo, hi in zip(ptr[:-1], ptr[1:])]


def block_weights(a, blocks, axis: str, csr=None, csc=None) -> np.ndarray:
    """||block||_F^2 as the reference computes it (matrix.py:170-189): BLAS
    dot of the C-order flattening of a dense block; for sparse storage the
    dot of the CSR (rows) / CSC (columns) value slices."""
    out = []
    for blk in blocks:
        s = _sel(blk)
        if csr is None:
            sub = a[s, :] if axis == "row" else a[:, s]
            flat = np.ravel(sub)
            out.append(float(flat @ flat))
            continue
        store = csr if axis == "row" else csc
        if isinstance(s, slice):
            chunk = store.data[store.indptr[s.start]:store.indptr[s.stop]]
            out.append(float(chunk @ chunk))
        else:
            tot = 0.0
            for i in s:
                chunk = store.data[store.indptr[i]:store.indptr[i + 1]]
                tot += float(chunk @ chunk)
            out.append(tot)
    return np.asarray(out)


class Sampler:
    def __init__(self, weights: np.ndarray):
        self.weights = np.asarray(weights, dtype=np.float64)
        if np.any(self.weights <= 0.0):
            raise ValueError("zero-weight entry: it could never be selected")
        self.cumulative = np.cumsum(self.weights)
        self.total = float(self.cumulative[-1])

    def sample(self, rng) -> int:
        v = rng.uniform() * self.total
        i = int(np.searchsorted(self.cumulative, v, side="right"))
        return min(i, self.weights.size - 1)


# -- the iteration (solvers.py:283-342) and the run loop (solvers.py:425-474) ----

class OracleSolver:
    """REBK / REK / RABK / RK / DSBGS on partitions given by block pointers
    or index blocks."""

    def __init__(self, a: np.ndarray, b: np.ndarray, row_blocks, col_blocks=None, alpha: float = 1.0,
                 algorithm: str = "rebk"):
        """row_blocks / col_blocks: block pointers (int array of length
        nb+1) or a list of index blocks (ranges or int arrays).  `a` is a
        dense array or a scipy sparse matrix (CSR + CSC twin, as the
        reference stores it, matrix.py:46-58)."""
        import scipy.sparse as sp

        self.sparse = sp.issparse(a)
        if self.sparse:
            csr = sp.csr_matrix(a, dtype=np.float64, copy=True)
            csr.sum_duplicates()
            csr.eliminate_zeros()
            csr.sort_indices()
            self.csr, self.csc = csr, csr.tocsc()
            self.a = None
        else:
            self.csr = self.csc = None
            self.a = np.ascontiguousarray(a, dtype=np.float64)
        self.b = np.asarray(b, dtype=np.float64)
        self.algorithm = algorithm
        self.extended = algorithm in ("rebk", "rek")
        self.dsbgs = algorithm == "dsbgs"
        if isinstance(row_blocks, np.ndarray) and row_blocks.dtype != object:
            row_blocks = blocks_from_ptr(row_blocks)
        self.row_sel = [_sel(bk) for bk in row_blocks]
        if self.sparse:
            self.row_blocks = [self.csr[s, :] for s in self.row_sel]
        else:
            self.row_blocks = [self.a[s, :] for s in self.row_sel]
        self.row_sampler = Sampler(block_weights(self.a, row_blocks, "row", self.csr, self.csc))
        self.row_scales = [float(alpha / w) for w in self.row_sampler.weights]
        self.b_blocks = [self.b[s] for s in self.row_sel]
        if self.extended or self.dsbgs:
            if isinstance(col_blocks, np.ndarray) and col_blocks.dtype != object:
                col_blocks = blocks_from_ptr(col_blocks)
            self.col_sel = [_sel(bk) for bk in col_blocks]
            if self.sparse:
                self.col_blocks = [self.csc[:, s] for s in self.col_sel]
            else:
                self.col_blocks = [self.a[:, s] for s in self.col_sel]
            self.col_sampler = Sampler(block_weights(self.a, col_blocks, "col", self.csr, self.csc))
            self.col_scales = [float(alpha / w) for w in self.col_sampler.weights]
        if self.dsbgs:
            self._dsbgs_tables(alpha)

    def _dsbgs_tables(self, alpha):
        """_build_dsbgs_tables (solvers.py:204-229): weight of every
        submatrix A[I_i, J_j] by the dot of its C-order flattening (sparse:
        of its CSR values), per column block the conditional sampler over
        the row blocks whose submatrix is nonzero, scales alpha / w."""
        s, t = len(self.row_blocks), len(self.col_sel)
        self.sub = [[None] * t for _ in range(s)]
        w = np.zeros((s, t))
        for i in range(s):
            for j, cs in enumerate(self.col_sel):
                sub = self.row_blocks[i][:, cs]
                self.sub[i][j] = sub
                if self.sparse:
                    w[i, j] = float(sub.data @ sub.data) if sub.nnz else 0.0
                else:
                    flat = np.ravel(sub)
                    w[i, j] = float(flat @ flat)
        self.ds_scales = [[float(alpha / v) if v > 0.0 else None for v in row] for row in w]
        self.ds_cond = []
        for j in range(t):
            alive = np.flatnonzero(w[:, j] > 0.0)
            self.ds_cond.append((Sampler(w[alive, j]), alive))

    def draw(self, rng) -> tuple[int, int]:
        """The two draws of one iteration (solvers.py:8-12, :373-375)."""
        if self.dsbgs:
            j = self.col_sampler.sample(rng)
            cond, alive = self.ds_cond[j]
            return j, int(alive[cond.sample(rng)])
        if self.extended:
            j = self.col_sampler.sample(rng)
        else:
            rng.uniform()
            j = -1
        return j, self.row_sampler.sample(rng)

    def picks(self, rng, count: int) -> np.ndarray:
        out = np.empty((count, 2), dtype=np.int64)
        if self.dsbgs:
            for k in range(count):
                out[k] = self.draw(rng)
            return out
        for k in range(count):
            if self.extended:
                out[k, 0] = self.col_sampler.sample(rng)
            else:
                rng.uniform()
                out[k, 0] = -1
            out[k, 1] = self.row_sampler.sample(rng)
        return out

    def step(self, x: np.ndarray, z: np.ndarray | None, j: int, i: int) -> None:
        if self.dsbgs:                        # step_dsbgs, solvers.py:371-381
            r = self.row_blocks[i] @ x
            r -= self.b_blocks[i]
            u = self.sub[i][j].T @ r
            x[self.col_sel[j]] -= self.ds_scales[i][j] * u
            return
        if self.extended:
            blk = self.col_blocks[j]          # _weighted_col_update, solvers.py:283-286
            u = blk.T @ z
            z -= self.col_scales[j] * (blk @ u)
        blk = self.row_blocks[i]              # _weighted_row_update, solvers.py:289-295
        r = blk @ x
        r -= self.b_blocks[i]
        if self.extended:
            r += z[self.row_sel[i]]
        x -= self.row_scales[i] * (blk.T @ r)

    def run(self, seed: int, max_iters: int, tol: float, x_star=None, stride: int = 1,
            mode: str = "oracle_error", x0=None, z0=None, rng=None, record: bool = False):
        """run() of solvers.py:425-474; returns a dict with the trace fields,
        the final iterates and the pick sequence."""
        rng = rng if rng is not None else OracleRng(seed)
        shape = self.csr.shape if self.sparse else self.a.shape
        x = np.zeros(shape[1]) if x0 is None else np.array(x0, dtype=np.float64)
        z = None
        if self.extended:
            z = self.b.copy() if z0 is None else np.array(z0, dtype=np.float64)
        xs = None if x_star is None else np.asarray(x_star, dtype=np.float64)
        fro = self.csr.data if self.sparse else self.a.ravel()
        scale = float(np.sqrt(float(fro @ fro)) * np.linalg.norm(self.b)) or 1.0
        mat, matT = (self.csr, self.csc.T) if self.sparse else (self.a, self.a.T)

        def err_of():
            if mode == "oracle_error":
                return float(np.linalg.norm(x - xs))
            if mode == "residual_proxy":
                r = mat @ x - self.b
                if z is not None:
                    r += z
                return float(np.linalg.norm(matT @ r)) / scale
            return None

        errors, ckpts, picks = [], [], []

        def check(k):
            e = err_of()
            if e is None:
                return None, False
            if record:
                errors.append(e)
                ckpts.append(k)
            return e, e <= tol

        final, conv = check(0)
        iters = 0
        t0 = time.perf_counter()
        if not conv:
            for k in range(1, max_iters + 1):
                j, i = self.draw(rng)
                picks.append((j, i))
                self.step(x, z, j, i)
                if k % stride == 0:
                    e, done = check(k)
                    final = e
                    if done:
                        conv, iters = True, k
                        break
            else:
                iters = max_iters
                if mode != "max_iters_only" and max_iters % stride != 0:
                    final, conv = check(max_iters)
        wall = time.perf_counter() - t0
        return dict(iters=iters, converged=conv, final_error=final, wall_time=wall, x=x, z=z,
                    picks=np.asarray(picks, dtype=np.int64).reshape(-1, 2),
                    errors=np.asarray(errors), checkpoints=np.asarray(ckpts, dtype=np.int64))

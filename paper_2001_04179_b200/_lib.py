"""ctypes binding of librebk.so (the C ABI declared in include/rebk.h).

The shared library is built in-tree (``paper_2001_04179_b200/librebk.so``,
see :mod:`paper_2001_04179_b200.build`).  There is deliberately no fallback:
if the library is missing or no CUDA device is present, the solver entry
points raise instead of computing anything on the CPU.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

LIB_PATH = os.environ.get("REBK_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "librebk.so")

REBK_OK = 0
ABI_VERSION = 2  # include/rebk.h REBK_ABI_VERSION (struct layouts below)
ERRORS = {
    -1: "REBK_EINVAL",
    -2: "REBK_ECUDA",
    -3: "REBK_ENOMEM",
    -4: "REBK_ENODEV",
    -5: "REBK_ENONFINITE",
}

ALGO_CODES = {"rebk": 0, "rek": 1, "rabk": 2, "rk": 3, "dsbgs": 4}
STOP_CODES = {"oracle_error": 0, "residual_proxy": 1, "max_iters_only": 2}


class RebkCfg(ctypes.Structure):
    _fields_ = [
        ("algorithm", c_int32),
        ("stop_mode", c_int32),
        ("tol", c_double),
        ("check_stride", c_int64),
        ("max_iters", c_int64),
        ("philox_key", c_uint64 * 2),
        ("draw_offset", c_uint64),
        ("n_row_blocks", c_int64),
        ("row_ptr", POINTER(c_int64)),
        ("row_cum", POINTER(c_double)),
        ("row_total", c_double),
        ("row_scale", POINTER(c_double)),
        ("n_col_blocks", c_int64),
        ("col_ptr", POINTER(c_int64)),
        ("col_cum", POINTER(c_double)),
        ("col_total", c_double),
        ("col_scale", POINTER(c_double)),
        ("picks", POINTER(c_int32)),
        ("record_errors", c_int32),
        ("grid_ctas", c_int32),
        ("residual_scale", c_double),
        ("nonfinite_stop", c_int32),
        ("reserved0", c_int32),
        ("dsbgs_off", POINTER(c_int64)),
        ("dsbgs_cum", POINTER(c_double)),
        ("dsbgs_total", POINTER(c_double)),
        ("dsbgs_alive", POINTER(c_int32)),
        ("dsbgs_scale", POINTER(c_double)),
    ]


class RebkShardRunArgs(ctypes.Structure):
    _fields_ = [
        ("max_iters", c_int64),
        ("stride", c_int64),
        ("tol", c_double),
        ("chunk", c_int32),
        ("extended", c_int32),
        ("picks", POINTER(c_int32)),
        ("n_col_blocks", c_int64),
        ("col_ptr", POINTER(c_int64)),
        ("col_scale", POINTER(c_double)),
        ("n_row_blocks", c_int64),
        ("row_ptr", POINTER(c_int64)),
        ("row_scale", POINTER(c_double)),
        ("local_ranges", POINTER(c_int64)),
        ("local_rows_dev", c_void_p),
        ("b_dev", c_void_p),
        ("x_dev", c_void_p),
        ("z_dev", c_void_p),
        ("xs_dev", c_void_p),
        ("n_picks", c_int64),
    ]


class RebkMmMatrix(ctypes.Structure):
    _fields_ = [
        ("rows", c_int64),
        ("cols", c_int64),
        ("dense", c_int32),
        ("reserved", c_int32),
        ("nnz", c_int64),
        ("indptr", POINTER(c_int64)),
        ("indices", POINTER(c_int32)),
        ("values", POINTER(c_double)),
        ("err_line", c_int64),
    ]


class RebkTrace(ctypes.Structure):
    _fields_ = [
        ("iters", c_int64),
        ("converged", c_int32),
        ("has_error", c_int32),
        ("final_error", c_double),
        ("loop_ms", c_double),
        ("errors", POINTER(c_double)),
        ("errors_cap", c_int64),
        ("n_checks", c_int64),
        ("grid_ctas", c_int32),
        ("kernel_path", c_int32),
        ("nonfinite_at", c_int64),
    ]


# every symbol include/rebk.h declares, with its ctypes signature
_P_D = POINTER(c_double)
_P_I64 = POINTER(c_int64)
SIGNATURES = {
    "rebk_abi_version": (c_int, []),
    "rebk_abi_struct_sizes": (c_int, [_P_I64, _P_I64, _P_I64]),
    "rebk_last_error": (c_char_p, []),
    "rebk_device_count": (c_int, [POINTER(c_int)]),
    "rebk_ctx_create_dense": (c_int, [_P_D, c_int64, c_int64, c_int64, c_int, POINTER(c_void_p)]),
    "rebk_ctx_create_dense_device": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int, POINTER(c_void_p)]),
    "rebk_ctx_create_csr": (c_int, [_P_I64, POINTER(c_int32), _P_D, c_int64, c_int64, c_int64, c_int,
                                    POINTER(c_void_p)]),
    "rebk_ctx_create_dense_f32": (c_int, [POINTER(ctypes.c_float), c_int64, c_int64, c_int64, c_int,
                                          POINTER(c_void_p)]),
    "rebk_run_mrhs": (c_int, [c_void_p, POINTER(RebkCfg), c_int64, POINTER(ctypes.c_float), POINTER(ctypes.c_float),
                              POINTER(ctypes.c_float), POINTER(ctypes.c_float), _P_D, POINTER(ctypes.c_float),
                              POINTER(ctypes.c_float), _P_I64, _P_D, POINTER(RebkTrace)]),
    "rebk_ctx_destroy": (c_int, [c_void_p]),
    "rebk_ctx_shape": (c_int, [c_void_p, _P_I64, _P_I64]),
    "rebk_run": (c_int, [c_void_p, POINTER(RebkCfg), _P_D, _P_D, _P_D, _P_D, _P_D, _P_D, POINTER(RebkTrace)]),
    "rebk_run_device": (c_int, [c_void_p, POINTER(RebkCfg), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                POINTER(RebkTrace)]),
    "rebk_shard_colstep": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "rebk_shard_zupdate": (c_int, [c_void_p, c_int64, c_int64, c_double, c_void_p, c_void_p, c_void_p]),
    "rebk_shard_rowstep": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "rebk_shard_xupdate": (c_int, [c_int64, c_double, c_void_p, c_void_p, c_void_p]),
    "rebk_shard_err2": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "rebk_shard_grid_ctas": (c_int, [c_int, POINTER(c_int)]),
    "rebk_shard_xchg_create": (c_int, [c_int, c_int, c_int64, c_int64, c_int, c_int, POINTER(c_void_p)]),
    "rebk_shard_xchg_ipc_handle": (c_int, [c_void_p, ctypes.c_char_p]),
    "rebk_shard_xchg_open_peers": (c_int, [c_void_p, ctypes.c_char_p]),
    "rebk_shard_xchg_probe": (c_int, [c_void_p, c_int, ctypes.c_uint64, POINTER(c_int)]),
    "rebk_shard_xchg_destroy": (c_int, [c_void_p]),
    "rebk_shard_run_device": (c_int, [c_void_p, c_void_p, POINTER(RebkCfg), _P_I64, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, POINTER(RebkTrace)]),
    "rebk_shard_run_virtual": (c_int, [c_void_p, c_int, _P_I64, _P_I64, POINTER(RebkCfg), c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_void_p, POINTER(RebkTrace)]),
    "rebk_sample_sequence": (c_int, [POINTER(RebkCfg), c_int64, c_int64, POINTER(c_int32)]),
    "rebk_block_frobenius_sq": (c_int, [c_void_p, c_int, c_int64, _P_I64, _P_D]),
    "rebk_block_sigma1_sq": (c_int, [c_void_p, c_int, c_int64, _P_I64, c_int, _P_D, POINTER(c_int32)]),
    "rebk_nccl_get_unique_id": (c_int, [c_char_p, ctypes.c_char_p]),
    "rebk_nccl_comm_create": (c_int, [c_char_p, ctypes.c_char_p, c_int, c_int, c_int, POINTER(c_void_p)]),
    "rebk_nccl_comm_destroy": (c_int, [c_void_p]),
    "rebk_shard_run": (c_int, [c_void_p, c_void_p, POINTER(RebkShardRunArgs), _P_I64, POINTER(c_int32), _P_D]),
    "rebk_philox_key": (c_int, [POINTER(c_uint32), c_int64, POINTER(c_uint32), c_int64, POINTER(c_uint64)]),
    "rebk_philox_uniforms_host": (c_int, [POINTER(c_uint64), c_uint64, c_int64, _P_D]),
    "rebk_mm_read": (c_int, [c_char_p, c_double, c_int, POINTER(RebkMmMatrix)]),
    "rebk_mm_free": (None, [POINTER(RebkMmMatrix)]),
    "rebk_host_gather_col_blocks": (c_int, [_P_D, c_int64, c_int64, c_int64, c_int64, _P_I64, _P_D, c_int]),
}

_lib = None


class RebkError(RuntimeError):
    """A failure reported by librebk (CUDA error, missing device, ...)."""


class NonFiniteError(RebkError):
    """REBK_ENONFINITE: a stopping reduction met NaN/Inf and the run was
    configured to stop there (rebk_cfg.nonfinite_stop)."""


def load() -> ctypes.CDLL:
    """Load librebk.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RebkError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.rebk_abi_version() != ABI_VERSION:
        raise RebkError(f"{LIB_PATH} has ABI {lib.rebk_abi_version()}, this binding expects {ABI_VERSION}: rebuild it")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != REBK_OK:
        msg = load().rebk_last_error().decode(errors="replace")
        code = ERRORS.get(rc, str(rc))
        if rc == -5:
            raise NonFiniteError(f"{what}: {msg}")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise RebkError(f"{what} failed ({code}): {msg}")


def device_count() -> int:
    lib = load()
    c = c_int(0)
    rc = lib.rebk_device_count(ctypes.byref(c))
    return c.value if rc == REBK_OK else 0


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(_P_D)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_P_I64)


def int_to_words(value: int) -> list[int]:
    """Little-endian uint32 digits of a non-negative int (0 -> [0]), the
    coercion numpy's SeedSequence applies to seeds and spawn keys."""
    value = int(value)
    if value < 0:
        raise ValueError("expected a non-negative integer")
    if value == 0:
        return [0]
    words = []
    while value > 0:
        words.append(value & 0xFFFFFFFF)
        value >>= 32
    return words


def philox_key(seed: int, spawn_key: tuple[int, ...] = ()) -> tuple[int, int]:
    """Philox key of Rng(seed, spawn_key) (sampling.py:33-37), computed by
    the library's restatement of numpy SeedSequence."""
    lib = load()
    ent = np.asarray(int_to_words(seed), dtype=np.uint32)
    spawn = []
    for k in spawn_key:
        spawn.extend(int_to_words(k))
    sp = np.asarray(spawn, dtype=np.uint32)
    out = (c_uint64 * 2)()
    rc = lib.rebk_philox_key(
        ent.ctypes.data_as(POINTER(c_uint32)), ent.size,
        sp.ctypes.data_as(POINTER(c_uint32)) if sp.size else None, sp.size, out,
    )
    check(rc, "rebk_philox_key")
    return int(out[0]), int(out[1])


def philox_uniforms_host(key: tuple[int, int], first: int, count: int) -> np.ndarray:
    lib = load()
    k = (c_uint64 * 2)(*key)
    out = np.empty(count, dtype=np.float64)
    check(lib.rebk_philox_uniforms_host(k, first, count, dptr(out)), "rebk_philox_uniforms_host")
    return out

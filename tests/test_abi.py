"""The C-ABI library loads and exports every symbol include/rebk.h declares;
host-only helpers agree with numpy; device entry points fail loudly (not
silently on the CPU) when there is no GPU.  No GPU needed."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2001_04179_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "rebk.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rebk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures out of sync with rebk.h"


def test_abi_version():
    assert _lib.load().rebk_abi_version() == _lib.ABI_VERSION == 2


def test_struct_layout_matches_header():
    # rebk_cfg / rebk_trace / rebk_shard_run_args: the ctypes mirrors have the
    # sizes the compiled C side uses
    sizes = [ctypes.c_int64() for _ in range(3)]
    assert _lib.load().rebk_abi_struct_sizes(*[ctypes.byref(s) for s in sizes]) == 0
    assert [s.value for s in sizes] == [ctypes.sizeof(_lib.RebkCfg), ctypes.sizeof(_lib.RebkTrace),
                                        ctypes.sizeof(_lib.RebkShardRunArgs)]
    assert ctypes.sizeof(_lib.RebkCfg) == 4 + 4 + 8 + 8 + 8 + 16 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 4 + 4 + 8 + 4 + 4 + 5 * 8
    assert ctypes.sizeof(_lib.RebkTrace) == 8 + 4 + 4 + 8 + 8 + 8 + 8 + 8 + 4 + 4 + 8


@pytest.mark.parametrize("seed,spawn", [(0, ()), (17, ()), (2024, ()), (2**64 + 3, ()), (4, (0,)),
                                        (4, (1, 2)), (2**40 + 1, (3, 5)), (12345678901234567890123, (7,))])
def test_philox_key_matches_numpy_seedsequence(seed, spawn):
    want = np.random.SeedSequence(seed, spawn_key=spawn).generate_state(2, np.uint64)
    assert _lib.philox_key(seed, spawn) == (int(want[0]), int(want[1]))


def test_host_philox_stream_matches_numpy_generator():
    for seed in (0, 5, 2024):
        g = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
        want = g.random(1001)
        got = _lib.philox_uniforms_host(_lib.philox_key(seed), 0, 1001)
        assert np.array_equal(got, want)
        # arbitrary offsets: draw d = word d%4 of block d//4
        got2 = _lib.philox_uniforms_host(_lib.philox_key(seed), 333, 50)
        assert np.array_equal(got2, want[333:383])


def test_reference_pinned_values_through_c_helper():
    got = _lib.philox_uniforms_host(_lib.philox_key(2024), 0, 3)
    assert got.tolist() == [0.2706129375647399, 0.6189835150824522, 0.038714373390908996]


def test_argument_errors_are_einval():
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.rebk_ctx_create_dense(None, 2, 2, 2, 0, ctypes.byref(h))
    assert rc == -1
    assert b"null" in lib.rebk_last_error()
    # device beta_max: argument checks happen before any device work
    ptr = np.array([0, 2], dtype=np.int64)
    out = np.zeros(1)
    rc = lib.rebk_block_sigma1_sq(None, 0, 1, _lib.i64ptr(ptr), 0, _lib.dptr(out), None)
    assert rc == -1 and b"bad argument" in lib.rebk_last_error()
    rc = lib.rebk_block_sigma1_sq(None, 2, 1, _lib.i64ptr(ptr), 0, _lib.dptr(out), None)
    assert rc == -1


@pytest.mark.skipif(_lib.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_device_fails_loudly():
    lib = _lib.load()
    a = np.eye(3)
    h = ctypes.c_void_p()
    rc = lib.rebk_ctx_create_dense(_lib.dptr(a), 3, 3, 3, 0, ctypes.byref(h))
    assert rc == -4  # REBK_ENODEV: no silent CPU path

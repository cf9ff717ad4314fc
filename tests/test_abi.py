"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every
symbol include/ee.h declares, and its pure host functions / argument
validation behave (no compute calls)."""

import ctypes

import numpy as np
import math
import os
import re

import pytest

import paper_2402_00518_b200 as ee
from oracle import ee_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ee.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ee_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    if not os.path.exists(ee.LIB_PATH):
        from paper_2402_00518_b200 import build
        build.build()
    lib = ee.load()
    names = _declared()
    assert "ee_tune_step" in names and "ee_init_heads" in names and "ee_adam_update" in names
    for n in names:
        assert hasattr(lib, n), n
    assert set(ee.EXPORTED) == set(names)


def test_lr_schedule_host_function_matches_oracle_pins():
    ee.load()
    T = 40000
    for it in (0, 1, 200, 400, 401, 20000, 39999, 40000):
        assert ee.ee_lr_at(it, T) == pytest.approx(O.lr_at(it, T), rel=1e-12, abs=1e-18)
    assert ee.ee_lr_at(400, T) == pytest.approx(1e-4)        # P:375 max
    assert ee.ee_lr_at(T, T) == pytest.approx(1e-5)          # P:375 min
    assert math.isnan(ee.ee_lr_at(T + 1, T))


def test_workspace_size_and_shape_validation():
    ee.load()
    c = ee.make_config(8192, 32000, 28672, 4, "mlp")
    ws = ee.ee_workspace_size(c, 65536)
    assert 20e9 < ws < 30e9                                   # ~23 GB at the 70B shape
    assert ee.ee_workspace_size(c, 0) < 1 << 20
    for bad in (ee.make_config(100, 512, 0, 1, "norm"),      # h not multiple of 64
                ee.make_config(128, 512, 100, 1, "mlp"),     # F not multiple of 128
                ee.make_config(128, 510, 0, 1, "norm"),      # V not multiple of 8
                ee.make_config(128, 512, 0, 0, "norm")):     # no exits
        with pytest.raises(ee.EEError):
            ee.ee_workspace_size(bad, 10)


def test_null_arguments_rejected_before_any_device_work():
    lib = ee.load()
    c = ee.make_config(128, 512, 0, 1, "norm")
    r = lib.ee_tune_step(ctypes.byref(c), None, 10, None, None, None, None, 0, None, None, None,
                         None, 0, None, None)
    assert r == 1                                             # EE_ERR_ARG
    assert b"NULL" in lib.ee_last_error()


@pytest.mark.parametrize("arch", ["embedding", "norm", "mlp", "layer"])
def test_dp_shard_layout_is_a_partition(arch):
    """ee_dp_shard_layout (host function of the fused DP path): every tensor's
    rows are covered exactly once by the P owners' row blocks, each rank's
    arena blocks are disjoint, in ee_head_tensors order, sized P x rows x C,
    and tile the arena; tensors the arch lacks own nothing."""
    ee.load()
    kw = dict(n_heads=2, n_kv_heads=1, seq_len=128) if arch == "layer" else {}
    h, V, F = 256, 1000, 384
    c = ee.make_config(h, V, F, 1, arch, **kw)
    shapes = ee.tensor_shapes(h, V, F, arch, c.n_kv_heads)
    for P in (1, 2, 3, 5, 8):
        for q in range(P):
            blocks = []
            for k in ee.TENSOR_NAMES:
                b, rows, off, total = ee.ee_dp_shard_layout(c, P, q, k)
                if k not in shapes:
                    assert rows == 0
                    continue
                C = shapes[k][-1]
                if rows:
                    blocks.append((off, off + P * rows * C))
            blocks.sort()
            pos = 0
            for lo, hi in blocks:
                assert lo == pos                               # contiguous, disjoint
                pos = hi
            assert pos == total
        for k, sh in shapes.items():
            R = 1 if len(sh) == 1 else sh[0]
            covered = []
            for q in range(P):
                b, rows, _, _ = ee.ee_dp_shard_layout(c, P, q, k)
                covered += list(range(b, b + rows))
            assert covered == list(range(R)), (P, k)
    with pytest.raises(ee.EEError):
        ee.ee_dp_shard_layout(c, 9, 0, "w_out")                # > EE_MAX_PEERS


def test_new_entry_points_reject_bad_arguments_without_a_gpu():
    """Argument validation of the peer-memory / fused-update entry points runs
    before any device work (synchronous EE_ERR_* codes)."""
    lib = ee.load()
    c = ee.make_config(128, 512, 256, 1, "mlp")
    ps = ee.ee_peer_set()
    ps.rank, ps.world = 0, 9                                   # > EE_MAX_PEERS
    assert lib.ee_peer_barrier(ctypes.byref(ps), 1, None, None) == 1
    ps.world = 1
    assert lib.ee_peer_barrier(ctypes.byref(ps), 1, None, None) == 1   # NULL workspace
    assert lib.ee_ipc_get_handle(None, None, None) == 1
    assert lib.ee_ipc_open(None, 0, None) == 1
    assert lib.ee_tune_step_rs(ctypes.byref(c), None, 10, None, None, None, None, None, None,
                               None, None, 0, None) == 1       # NULL grad arenas
    assert lib.ee_tune_step_adam(ctypes.byref(c), None, 10, None, None, None, None, None, None,
                                 1e-3, 0.9, 0.95, 1e-5, 0.0, 1, 1.0, None, None, None, None, 0,
                                 None) == 1                    # NULL parameter state
    assert lib.ee_vp_exit_backward_slots(ctypes.byref(c), None, 0, 0, None, None, 0, None, 0,
                                         None, None, 0, None) == 1   # n_slots = 0


@pytest.mark.parametrize("arch", ["embedding", "norm", "mlp", "layer"])
def test_comm_arena_size_and_create_without_a_gpu(arch):
    """ee_comm_* host logic (include/ee.h): the arena holds the barrier
    signals, the small reductions, two gradient arenas of the fused
    reduce-scatter (at least one full gradient set each) and, under VP, the
    all-gathered targets / z, the CE statistics and the dz slots; creation
    validates its arguments and never touches the device."""
    ee.load()
    h, V, F = 256, 1000, 384
    kw = dict(n_heads=2, n_kv_heads=1, seq_len=64) if arch == "layer" else {}
    c = ee.make_config(h, V, F, 2, arch, **kw)
    shapes = ee.tensor_shapes(h, V, F, arch, 1 if arch == "layer" else 0)
    full = sum(int(np.prod(s)) for s in shapes.values()) * 4
    for P in (1, 2, 3, 8):
        b = ee.ee_comm_arena_size(c, "dp", P, 128)
        assert b >= 2 * full
        bv = ee.ee_comm_arena_size(ee.make_config(h, V, F, 2, arch, 1e-5, 0, 504, **kw), "vp",
                                   P, 128)
        n_all = 128 * P
        assert bv >= n_all * (4 + 2 * h + 32)
    lib = ee.lib() if hasattr(ee, "lib") else ee.load()
    h_ = ctypes.c_void_p()
    fake = (ctypes.c_void_p * 2)(0x100000, 0x200000)
    b = ee.ee_comm_arena_size(c, "dp", 2, 128)
    assert lib.ee_comm_create(ctypes.byref(h_), ctypes.byref(c), 0, 2, 0, 128, fake, b) == 0
    assert lib.ee_comm_destroy(h_) == 0
    assert lib.ee_comm_create(ctypes.byref(h_), ctypes.byref(c), 0, 2, 2, 128, fake, b) == 1
    assert lib.ee_comm_create(ctypes.byref(h_), ctypes.byref(c), 0, 2, 0, 128, fake, b - 1) == 8
    bad = (ctypes.c_void_p * 2)(0x100010, 0x200000)                  # not 256-byte aligned
    assert lib.ee_comm_create(ctypes.byref(h_), ctypes.byref(c), 0, 2, 0, 128, bad, b) == 3
    shard = ee.make_config(h, V, F, 2, arch, 1e-5, 0, 504, **kw)      # DP needs full W_out
    assert lib.ee_comm_create(ctypes.byref(h_), ctypes.byref(shard), 0, 2, 0, 128, fake, b) == 1

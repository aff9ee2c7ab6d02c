"""Seeded fuzz of the C ABI's validation (include/lora.h: "validation is complete
and synchronous before any launch; errors return a status naming the offending
argument"), CPU only: random valid problems with exactly ONE injected fault
(bad dimension, rank > 64, NULL input, misaligned pointer, short workspace,
bad dropout p / offsets) must return that fault's status and a non-empty
message -- never crash, never reach the device; fault-free calls on this
GPU-less host must fail with LORA_ERR_CUDA / LORA_ERR_UNSUPPORTED (no CPU
fallback)."""
import ctypes

import numpy as np
import pytest

import paper_2403_11366_b200 as L

ALIGN_BASE = 1 << 32   # fake, never dereferenced, 16-byte aligned, disjoint regions


def _ptrs(k):
    return [ALIGN_BASE * (i + 1) for i in range(k)]


def _case(rng):
    T = int(rng.integers(1, 5000))
    n = 8 * int(rng.integers(1, 1500))
    m = 8 * int(rng.integers(1, 1500))
    r = int(rng.integers(1, 65))
    return T, n, m, r


FAULTS = ["none", "d_in", "d_out", "tokens", "rank0", "rank65", "alpha", "null_x", "misaligned_w0", "short_ws",
          "drop_p", "drop_col_offset"]


@pytest.mark.parametrize("seed", range(40))
def test_forward_single_fault(seed):
    rng = np.random.default_rng(seed)
    T, n, m, r = _case(rng)
    fault = FAULTS[seed % len(FAULTS)]
    alpha = 16.0
    if fault == "d_in":
        n = n + 4
    elif fault == "d_out":
        m = -8
    elif fault == "tokens":
        T = -1
    elif fault == "rank0":
        r = 0
    elif fault == "rank65":
        r = 65
    elif fault == "alpha":
        alpha = float("inf")
    d = L.dims(T, n, m, r, alpha)
    x, w0, a, b, y, ws = _ptrs(6)
    if fault == "null_x":
        x = None
    if fault == "misaligned_w0":
        w0 += 8
    need = (int(L.lib.lora_linear_fwd_dropout_workspace_bytes(ctypes.byref(d))) if fault.startswith("drop")
            else L.lora_linear_fwd_workspace_bytes(d))
    wsb = max(need, 1) - 1 if fault == "short_ws" else max(need, 1 << 20)
    if fault.startswith("drop"):
        dr = L.lora_dropout(2.0 if fault == "drop_p" else 0.1, 1, 2, None, None, 0, 12 if fault == "drop_col_offset" else 0)
        st = L.lib.lora_linear_fwd_dropout(ctypes.byref(d), ctypes.byref(dr), x, w0, a, b, None, y, None, ws, wsb, None)
    else:
        st = L.lib.lora_linear_fwd(ctypes.byref(d), x, w0, a, b, None, y, None, ws, wsb, None)
    expect = {"none": (4, 5), "d_in": (2,), "d_out": (2,), "tokens": (2,), "rank0": (2,), "rank65": (4,),
              "alpha": (1,), "null_x": (1,), "misaligned_w0": (3,), "short_ws": (7,), "drop_p": (1,),
              "drop_col_offset": (1,)}[fault]
    assert st in expect, (seed, fault, (T, n, m, r), st, L.lib.lora_last_error())
    assert L.lib.lora_last_error().decode()


@pytest.mark.parametrize("seed", range(24))
def test_backward_single_fault(seed):
    rng = np.random.default_rng(1000 + seed)
    T, n, m, r = _case(rng)
    faults = ["none", "null_dy", "misaligned_db", "short_ws", "accumulate", "alias_da_x"]
    fault = faults[seed % len(faults)]
    d = L.dims(T, n, m, r, 16.0)
    x, w0, a, b, dy, dx, da, db, ws = _ptrs(9)
    need = L.lora_linear_bwd_workspace_bytes(d)
    wsb = need - 1 if fault == "short_ws" else need
    acc = 2 if fault == "accumulate" else 0
    if fault == "null_dy":
        dy = None
    if fault == "misaligned_db":
        db += 4
    if fault == "alias_da_x":
        da = x
    st = L.lib.lora_linear_bwd(ctypes.byref(d), x, w0, a, b, None, dy, dx, da, db, acc, ws, wsb, None)
    expect = {"none": (4, 5), "null_dy": (1,), "misaligned_db": (3,), "short_ws": (7,), "accumulate": (1,),
              "alias_da_x": (1,)}[fault]
    assert st in expect, (seed, fault, (T, n, m, r), st, L.lib.lora_last_error())

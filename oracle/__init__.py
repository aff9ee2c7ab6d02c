"""CPU fp64 oracle for the LoRA-linear hot path (ctypes front of lora_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2403_11366_b200`` never imports it and
shares no code with it ("Oracle").

Every function follows PAPER.md Eq. 1 and the LoRA
paragraph in the row-vector orientation of DESIGN.md R1;
the arithmetic itself lives in ``lora_oracle.c`` (plain fp64 loops).

Parity pins for every function are in ``tests/test_oracle_pins.py``; none of
the oracle's outputs is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lora_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_u16p = ctypes.POINTER(ctypes.c_uint16)
_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile lora_oracle.c with gcc -O2 -fopenmp (no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.oracle_lora_fwd.argtypes = [
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
            _u16p, _u16p, _u16p, _u16p, _u16p, _i64p, ctypes.c_int64, _f64p, _f64p]
        lib.oracle_lora_fwd.restype = ctypes.c_int
        lib.oracle_lora_bwd.argtypes = [
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
            _u16p, _u16p, _u16p, _u16p, _u16p, _i64p, ctypes.c_int64, _f64p, _f64p, _f64p, _f64p]
        lib.oracle_lora_bwd.restype = ctypes.c_int
        lib.oracle_lora_merge.argtypes = [
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
            _u16p, _u16p, _u16p, _f64p]
        lib.oracle_lora_merge.restype = ctypes.c_int
        _u8p = ctypes.POINTER(ctypes.c_uint8)
        lib.oracle_lora_fwd_dropout.argtypes = [
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
            _u16p, _u16p, _u16p, _u16p, _u16p, _u8p, ctypes.c_double, _i64p, ctypes.c_int64, _f64p, _f64p]
        lib.oracle_lora_fwd_dropout.restype = ctypes.c_int
        lib.oracle_lora_bwd_dropout.argtypes = [
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
            _u16p, _u16p, _u16p, _u16p, _u16p, _u8p, ctypes.c_double, _i64p, ctypes.c_int64,
            _f64p, _f64p, _f64p, _f64p]
        lib.oracle_lora_bwd_dropout.restype = ctypes.c_int
        lib.oracle_philox4x32_10.argtypes = [ctypes.POINTER(ctypes.c_uint32)] * 3
        lib.oracle_philox4x32_10.restype = None
        lib.oracle_dropout_threshold.argtypes = [ctypes.c_float]
        lib.oracle_dropout_threshold.restype = ctypes.c_uint32
        lib.oracle_dropout_mask.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_float, ctypes.c_uint64,
                                            ctypes.c_uint64, _u8p]
        lib.oracle_dropout_mask.restype = ctypes.c_int
        lib.oracle_adam_step.argtypes = [ctypes.c_int64, _f64p, _f64p, _f64p, _f64p, ctypes.c_int64,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        lib.oracle_adam_step.restype = ctypes.c_int
        lib.oracle_scale.argtypes = [ctypes.c_int, ctypes.c_double]
        lib.oracle_scale.restype = ctypes.c_double
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _u16(a):
    if a is None:
        return None, None
    a = np.ascontiguousarray(a, dtype=np.uint16)
    return a, a.ctypes.data_as(_u16p)


def _rows(rows, T):
    if rows is None:
        return None, None, T
    r = np.ascontiguousarray(rows, dtype=np.int64)
    if r.size and (r.min() < 0 or r.max() >= T):
        raise ValueError("row index out of range")
    return r, r.ctypes.data_as(_i64p), int(r.size)


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(nt: int) -> None:
    _load().oracle_set_num_threads(int(nt))


def scale(r: int, alpha: float) -> float:
    """s = alpha / r (R2; Listing 3)."""
    return _load().oracle_scale(int(r), float(alpha))


def philox4x32_10(ctr, key):
    """Philox4x32-10 block (Salmon et al., SC'11) -> 4 uint32 words."""
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    _load().oracle_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def dropout_threshold(p: float) -> int:
    """floor(p 2^32) for the fp32 dropout probability p (keep iff word >= it)."""
    return int(_load().oracle_dropout_threshold(float(np.float32(p))))


def dropout_mask(T: int, n: int, p: float, seed: int, offset: int) -> np.ndarray:
    """LoRA-dropout keep mask M [T, n] uint8 (Listing 3 LORA_DROPOUT, PAPER.md:82;
    DESIGN.md R7): M[t,k] = Philox4x32-10((k/4, t, offset), seed)[k % 4] >= floor(p 2^32)."""
    mask = np.empty((T, n), np.uint8)
    rc = _load().oracle_dropout_mask(int(T), int(n), float(np.float32(p)), int(seed) & (2**64 - 1),
                                     int(offset) & (2**64 - 1), mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    if rc != 0:
        raise ValueError(f"oracle_dropout_mask failed rc={rc}")
    return mask


def _dropout_args(dropout, T, n):
    """dropout = (p, seed, offset) -> (mask [T, n] uint8, q = 1 / (1 - p)); p is taken as fp32."""
    p, seed, offset = dropout
    p32 = float(np.float32(p))
    mask = dropout_mask(T, n, p32, seed, offset)
    return mask, 1.0 / (1.0 - p32)


def lora_fwd(x, w0, a, b, alpha, bias=None, rows=None, dropout=None):
    """Eq. 1 line 1: y = x W0^T + s (x A^T) B^T (+ b0).

    All tensor arguments are bf16 bit patterns (uint16).  ``rows`` selects the
    tokens to evaluate (None: all).  ``dropout = (p, seed, offset)`` applies
    LoRA dropout to the adapter input (R7).  Returns (y [n_rows, m],
    h [n_rows, r]) in float64.
    """
    T, n = x.shape
    m, r = b.shape
    assert w0.shape == (m, n) and a.shape == (r, n)
    if bias is not None:
        assert bias.shape == (m,)
    xs, xp = _u16(x); ws, wp = _u16(w0); as_, ap = _u16(a); bs, bp = _u16(b)
    bis, bip = _u16(bias)
    rs, rp, nr = _rows(rows, T)
    y = np.empty((nr, m), np.float64)
    h = np.empty((nr, r), np.float64)
    if dropout is None:
        rc = _load().oracle_lora_fwd(T, n, m, r, float(alpha), xp, wp, ap, bp, bip, rp, nr,
                                     y.ctypes.data_as(_f64p), h.ctypes.data_as(_f64p))
    else:
        mask, q = _dropout_args(dropout, T, n)
        rc = _load().oracle_lora_fwd_dropout(T, n, m, r, float(alpha), xp, wp, ap, bp, bip,
                                             mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), q, rp, nr,
                                             y.ctypes.data_as(_f64p), h.ctypes.data_as(_f64p))
    if rc != 0:
        raise ValueError(f"oracle_lora_fwd failed rc={rc}")
    return y, h


def lora_bwd(x, w0, a, b, dy, alpha, rows=None, want_dx=True, dropout=None):
    """Backward of Eq. 1 for A, B trainable; ``dropout`` as in lora_fwd.

    Returns dict with dx [n_rows, n] (or None), gh [T, r], da [r, n], db [m, r]
    in float64.
    """
    T, n = x.shape
    m, r = b.shape
    assert w0.shape == (m, n) and a.shape == (r, n) and dy.shape == (T, m)
    xs, xp = _u16(x); ws, wp = _u16(w0); as_, ap = _u16(a); bs, bp = _u16(b)
    gs, gp = _u16(dy)
    rs, rp, nr = _rows(rows, T)
    dx = np.empty((nr, n), np.float64) if want_dx else None
    gh = np.empty((T, r), np.float64)
    da = np.empty((r, n), np.float64)
    db = np.empty((m, r), np.float64)
    outs = (dx.ctypes.data_as(_f64p) if dx is not None else None,
            gh.ctypes.data_as(_f64p), da.ctypes.data_as(_f64p), db.ctypes.data_as(_f64p))
    if dropout is None:
        rc = _load().oracle_lora_bwd(T, n, m, r, float(alpha), xp, wp, ap, bp, gp, rp, nr, *outs)
    else:
        mask, q = _dropout_args(dropout, T, n)
        rc = _load().oracle_lora_bwd_dropout(T, n, m, r, float(alpha), xp, wp, ap, bp, gp,
                                             mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), q, rp, nr,
                                             *outs)
    if rc != 0:
        raise ValueError(f"oracle_lora_bwd failed rc={rc}")
    return {"dx": dx, "gh": gh, "da": da, "db": db}


def lora_merge(w0, a, b, alpha):
    """Eq. 1 line 2: W' = W0 + s B A, float64 [m, n]."""
    m, n = w0.shape
    r = a.shape[0]
    assert a.shape == (r, n) and b.shape == (m, r)
    ws, wp = _u16(w0); as_, ap = _u16(a); bs, bp = _u16(b)
    out = np.empty((m, n), np.float64)
    rc = _load().oracle_lora_merge(n, m, r, float(alpha), wp, ap, bp, out.ctypes.data_as(_f64p))
    if rc != 0:
        raise ValueError(f"oracle_lora_merge failed rc={rc}")
    return out


def adam_step(theta, grad, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    """One bias-corrected Adam step (Kingma & Ba 2015, Alg. 1) in
    fp64.  Returns new (theta, m, v) arrays (inputs are not modified)."""
    th = np.array(theta, np.float64, copy=True).ravel()
    g = np.ascontiguousarray(grad, np.float64).ravel()
    mm = np.array(m, np.float64, copy=True).ravel()
    vv = np.array(v, np.float64, copy=True).ravel()
    assert th.size == g.size == mm.size == vv.size
    rc = _load().oracle_adam_step(th.size, th.ctypes.data_as(_f64p), g.ctypes.data_as(_f64p),
                                  mm.ctypes.data_as(_f64p), vv.ctypes.data_as(_f64p), int(t), float(lr), float(b1),
                                  float(b2), float(eps))
    if rc != 0:
        raise ValueError(f"oracle_adam_step failed rc={rc}")
    shape = np.shape(theta)
    return th.reshape(shape), mm.reshape(shape), vv.reshape(shape)

"""paper_2403_11366_b200 -- B200-native LoRA-linear hot path of JORA (arXiv 2403.11366).

Thin Python binding over the C ABI of ``liblora.so`` (``include/lora.h``).
It only marshals arguments (torch tensors -> device pointers, the current
CUDA stream) -- every step of the path runs in the sm_100a kernels of
``csrc/``.  There is no CPU fallback: if the library is missing, importing
this package raises, and every call on a non-B200 device returns an error.

Functions keep the C names:
    lora_linear_fwd   y = x W0^T + s (x A^T) B^T (+ b0)   (Eq. 1, :117)
    lora_linear_bwd   dx, dA, dB (A, B trainable, W0 frozen)
    lora_merge        W0 + s B A                           (Eq. 1 line 2, :118)
with s = alpha / r (Listing 3).
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

__all__ = [
    "LoraError", "lora_dims", "lib", "lora_linear_fwd", "lora_linear_bwd", "lora_merge",
    "lora_linear_fwd_workspace_bytes", "lora_linear_bwd_workspace_bytes",
    "lora_last_launch_count", "lora_device_check", "LIB_PATH", "header_functions",
]

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LORA_LIB_PATH") or os.path.join(_PKG, "liblora.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG), "include", "lora.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2403_11366_b200.build` "
        "(there is no CPU fallback for the LoRA hot path)")

lib = ctypes.CDLL(LIB_PATH)


class lora_dims(ctypes.Structure):
    _fields_ = [("tokens", ctypes.c_int64), ("d_in", ctypes.c_int64), ("d_out", ctypes.c_int64),
                ("rank", ctypes.c_int32), ("alpha", ctypes.c_float)]


class lora_fwd_problem(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("w0", ctypes.c_void_p), ("a", ctypes.c_void_p), ("b", ctypes.c_void_p),
                ("bias", ctypes.c_void_p), ("y", ctypes.c_void_p), ("h_out", ctypes.c_void_p)]


class lora_bwd_problem(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("w0", ctypes.c_void_p), ("a", ctypes.c_void_p), ("b", ctypes.c_void_p),
                ("h_saved", ctypes.c_void_p), ("dy", ctypes.c_void_p), ("dx", ctypes.c_void_p),
                ("da", ctypes.c_void_p), ("db", ctypes.c_void_p)]


class lora_adam_tensor(ctypes.Structure):
    _fields_ = [("param", ctypes.c_void_p), ("master", ctypes.c_void_p), ("grad", ctypes.c_void_p),
                ("m", ctypes.c_void_p), ("v", ctypes.c_void_p), ("numel", ctypes.c_int64)]


class lora_adam_hparams(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float)]


LORA_ADAM_MAX_TENSORS = 64


class lora_dropout(ctypes.Structure):
    _fields_ = [("p", ctypes.c_float), ("seed", ctypes.c_uint64), ("offset", ctypes.c_uint64),
                ("keep_bits", ctypes.c_void_p), ("masked_x", ctypes.c_void_p),
                ("row_offset", ctypes.c_int64), ("col_offset", ctypes.c_int64)]


LORA_MAX_GROUP = 8
_vp = ctypes.c_void_p
_fp = ctypes.c_void_p  # float* passed as raw address
_dp = ctypes.POINTER(lora_dims)
_st = ctypes.c_int

lib.lora_linear_fwd_workspace_bytes.argtypes = [_dp]
lib.lora_linear_fwd_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_bwd_workspace_bytes.argtypes = [_dp]
lib.lora_linear_bwd_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_fwd.argtypes = [_dp, _vp, _vp, _vp, _vp, _vp, _vp, _fp, _vp, ctypes.c_size_t, _vp]
lib.lora_linear_fwd.restype = _st
lib.lora_linear_bwd.argtypes = [_dp, _vp, _vp, _vp, _vp, _fp, _vp, _vp, _fp, _fp, ctypes.c_int,
                                _vp, ctypes.c_size_t, _vp]
_drp = ctypes.POINTER(lora_dropout)
lib.lora_linear_fwd_dropout_workspace_bytes.argtypes = [_dp]
lib.lora_linear_fwd_dropout_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_bwd_dropout_workspace_bytes.argtypes = [_dp]
lib.lora_linear_bwd_dropout_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_fwd_dropout.argtypes = [_dp, _drp, _vp, _vp, _vp, _vp, _vp, _vp, _fp, _vp, ctypes.c_size_t, _vp]
lib.lora_linear_fwd_dropout.restype = ctypes.c_int
lib.lora_linear_bwd_dropout.argtypes = [_dp, _drp, _vp, _vp, _vp, _vp, _fp, _vp, _vp, _fp, _fp, ctypes.c_int,
                                        _vp, ctypes.c_size_t, _vp]
lib.lora_linear_bwd_dropout.restype = ctypes.c_int
lib.lora_adam_step.argtypes = [ctypes.c_int, ctypes.POINTER(lora_adam_tensor), ctypes.POINTER(lora_adam_hparams),
                               ctypes.c_int64, _vp]
lib.lora_adam_step.restype = ctypes.c_int
lib.lora_dropout_mask.argtypes = [ctypes.c_int64, ctypes.c_int64, _drp, _vp, _vp]
lib.lora_dropout_mask.restype = ctypes.c_int
lib.lora_linear_bwd.restype = _st
lib.lora_linear_fwd_grouped_workspace_bytes.argtypes = [ctypes.c_int, _dp]
lib.lora_linear_fwd_grouped_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_bwd_grouped_workspace_bytes.argtypes = [ctypes.c_int, _dp]
lib.lora_linear_bwd_grouped_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_fwd_grouped.argtypes = [ctypes.c_int, _dp, ctypes.POINTER(lora_fwd_problem), _vp, ctypes.c_size_t,
                                        _vp]
lib.lora_linear_fwd_grouped.restype = _st
lib.lora_linear_bwd_grouped.argtypes = [ctypes.c_int, _dp, ctypes.POINTER(lora_bwd_problem), ctypes.c_int, _vp,
                                        ctypes.c_size_t, _vp]
lib.lora_linear_bwd_grouped.restype = _st
lib.lora_linear_fwd_grouped_dropout_workspace_bytes.argtypes = [ctypes.c_int, _dp]
lib.lora_linear_fwd_grouped_dropout_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_bwd_grouped_dropout_workspace_bytes.argtypes = [ctypes.c_int, _dp]
lib.lora_linear_bwd_grouped_dropout_workspace_bytes.restype = ctypes.c_size_t
lib.lora_linear_fwd_grouped_dropout.argtypes = [ctypes.c_int, _dp, _drp, ctypes.POINTER(lora_fwd_problem), _vp,
                                                ctypes.c_size_t, _vp]
lib.lora_linear_fwd_grouped_dropout.restype = _st
lib.lora_linear_bwd_grouped_dropout.argtypes = [ctypes.c_int, _dp, _drp, ctypes.POINTER(lora_bwd_problem),
                                                ctypes.c_int, _vp, ctypes.c_size_t, _vp]
lib.lora_linear_bwd_grouped_dropout.restype = _st
lib.lora_merge.argtypes = [_dp, _vp, _vp, _vp, _vp, _vp]
lib.lora_merge.restype = _st
lib.lora_status_string.argtypes = [_st]
lib.lora_status_string.restype = ctypes.c_char_p
lib.lora_last_error.restype = ctypes.c_char_p
lib.lora_version.restype = ctypes.c_int
lib.lora_device_check.restype = _st
lib.lora_last_launch_count.restype = ctypes.c_int
lib.lora_comm_unique_id.argtypes = [ctypes.c_char_p]
lib.lora_comm_unique_id.restype = _st
lib.lora_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_vp)]
lib.lora_comm_init.restype = _st
lib.lora_comm_destroy.argtypes = [_vp]
lib.lora_comm_destroy.restype = _st
lib.lora_comm_size.argtypes = [_vp]
lib.lora_comm_size.restype = ctypes.c_int
lib.lora_comm_rank.argtypes = [_vp]
lib.lora_comm_rank.restype = ctypes.c_int
lib.lora_allreduce.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int, _vp]
lib.lora_allreduce.restype = _st
lib.lora_tp_linear_fwd.argtypes = [_vp, ctypes.c_int, _dp, _vp, _vp, _vp, _vp, _vp, _vp, _fp, _vp,
                                   ctypes.c_size_t, _vp]
lib.lora_tp_linear_fwd.restype = _st
lib.lora_tp_linear_bwd_workspace_bytes.argtypes = [_dp]
lib.lora_tp_linear_bwd_workspace_bytes.restype = ctypes.c_size_t
lib.lora_tp_linear_bwd.argtypes = [_vp, ctypes.c_int, _dp, _vp, _vp, _vp, _vp, _fp, _vp, _vp, _fp, _fp,
                                   ctypes.c_int, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
lib.lora_tp_linear_bwd.restype = _st
lib.lora_tp_linear_bwd_column_group_dropout_workspace_bytes.argtypes = [ctypes.c_int, _dp]
lib.lora_tp_linear_bwd_column_group_dropout_workspace_bytes.restype = ctypes.c_size_t
lib.lora_tp_linear_bwd_column_group_dropout.argtypes = [_vp, ctypes.c_int, _dp, _drp,
                                                        ctypes.POINTER(lora_bwd_problem), _vp, ctypes.c_int,
                                                        ctypes.c_int, _vp, ctypes.c_size_t, _vp]
lib.lora_tp_linear_bwd_column_group_dropout.restype = _st
lib.lora_tp_linear_fwd_dropout.argtypes = [_vp, ctypes.c_int, _dp, _drp, _vp, _vp, _vp, _vp, _vp, _vp, _fp, _vp,
                                           ctypes.c_size_t, _vp]
lib.lora_tp_linear_fwd_dropout.restype = _st
lib.lora_tp_linear_bwd_dropout_workspace_bytes.argtypes = [_dp]
lib.lora_tp_linear_bwd_dropout_workspace_bytes.restype = ctypes.c_size_t
lib.lora_tp_linear_bwd_dropout.argtypes = [_vp, ctypes.c_int, _dp, _drp, _vp, _vp, _vp, _vp, _fp, _vp, _vp, _fp,
                                           _fp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
lib.lora_tp_linear_bwd_dropout.restype = _st
lib.lora_tp_linear_bwd_column_group_workspace_bytes.argtypes = [ctypes.c_int, _dp]
lib.lora_tp_linear_bwd_column_group_workspace_bytes.restype = ctypes.c_size_t
lib.lora_tp_linear_bwd_column_group.argtypes = [_vp, ctypes.c_int, _dp, ctypes.POINTER(lora_bwd_problem), _vp,
                                                ctypes.c_int, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
lib.lora_tp_linear_bwd_column_group.restype = _st

LORA_SYMM_HANDLE_BYTES = 64
lib.lora_symm_create.argtypes = [ctypes.c_size_t, ctypes.POINTER(_vp)]
lib.lora_symm_create.restype = _st
lib.lora_symm_ipc_handle.argtypes = [_vp, ctypes.c_char_p]
lib.lora_symm_ipc_handle.restype = _st
lib.lora_symm_connect.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
lib.lora_symm_connect.restype = _st
lib.lora_symm_connect_local.argtypes = [ctypes.c_int, ctypes.POINTER(_vp)]
lib.lora_symm_connect_local.restype = _st
lib.lora_symm_ptr.argtypes = [_vp]
lib.lora_symm_ptr.restype = _vp
lib.lora_symm_bytes.argtypes = [_vp]
lib.lora_symm_bytes.restype = ctypes.c_size_t
lib.lora_symm_last_placement.argtypes = [_vp]
lib.lora_symm_last_placement.restype = ctypes.c_int
lib.lora_symm_destroy.argtypes = [_vp]
lib.lora_symm_destroy.restype = _st
lib.lora_tp_linear_fwd_fused.argtypes = [_vp, _dp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, ctypes.c_size_t, _fp,
                                         _vp, ctypes.c_size_t, _vp]
lib.lora_tp_linear_fwd_fused.restype = _st
lib.lora_tp_linear_bwd_column_group_fused.argtypes = [_vp, _vp, ctypes.c_int, _dp, ctypes.POINTER(lora_bwd_problem),
                                                      ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, _vp,
                                                      ctypes.c_size_t, _vp]
lib.lora_tp_linear_bwd_column_group_fused.restype = _st

class lora_host_tensor(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("dtype", ctypes.c_int), ("ndim", ctypes.c_int),
                ("shape", ctypes.c_int64 * 4), ("data", ctypes.c_void_p)]


class lora_export_tensor(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("w0", ctypes.c_void_p), ("a", ctypes.c_void_p), ("b", ctypes.c_void_p),
                ("dims", lora_dims), ("dtype", ctypes.c_int), ("ndim", ctypes.c_int), ("shape", ctypes.c_int64 * 4)]


lib.lora_write_safetensors.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(lora_host_tensor)]
lib.lora_write_safetensors.restype = _st
lib.lora_export_merged.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(lora_export_tensor), _vp]
lib.lora_export_merged.restype = _st

_i64 = ctypes.c_int64
lib.lora_rmsnorm_fwd.argtypes = [_i64, _i64, ctypes.c_float, _vp, _vp, _vp, _vp, _vp, _fp, _vp]
lib.lora_rmsnorm_fwd.restype = _st
lib.lora_rmsnorm_bwd.argtypes = [_i64, _i64, _vp, _vp, _vp, _fp, _vp, _vp, _vp]
lib.lora_rmsnorm_bwd.restype = _st
lib.lora_rope.argtypes = [_i64, ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_float, ctypes.c_int, _vp, _vp]
lib.lora_rope.restype = _st
lib.lora_swiglu_fwd.argtypes = [_i64, _vp, _vp, _vp, _vp]
lib.lora_swiglu_fwd.restype = _st
lib.lora_swiglu_bwd.argtypes = [_i64, _vp, _vp, _vp, _vp, _vp, _vp]
lib.lora_swiglu_bwd.restype = _st
lib.lora_sum_bf16.argtypes = [_i64, ctypes.c_int, ctypes.POINTER(_vp), _vp, _vp]
lib.lora_sum_bf16.restype = _st

lib.lora_captured_sync_words_free.restype = ctypes.c_int
lib.lora_profile_next_bwd.argtypes = [ctypes.POINTER(_vp)]
lib.lora_profile_next_bwd.restype = _st

STATUS = {0: "LORA_OK", 1: "LORA_ERR_INVALID", 2: "LORA_ERR_SHAPE", 3: "LORA_ERR_ALIGN",
          4: "LORA_ERR_UNSUPPORTED", 5: "LORA_ERR_CUDA", 6: "LORA_ERR_NCCL", 7: "LORA_ERR_WORKSPACE"}


class LoraError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        msg = lib.lora_last_error().decode(errors="replace")
        super().__init__(f"{where}: {self.name}: {msg}")


def _check(st: int, where: str) -> None:
    if st != 0:
        raise LoraError(st, where)


def header_functions() -> list[str]:
    """Names of every function include/lora.h declares (for ABI tests)."""
    txt = open(HEADER_PATH).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lora_[a-z0-9_]+)\s*\(", txt)))


def dims(tokens: int, d_in: int, d_out: int, rank: int, alpha: float) -> lora_dims:
    return lora_dims(int(tokens), int(d_in), int(d_out), int(rank), float(alpha))


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _bf16(t, name, shape):
    if not (t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous CUDA bf16 tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _f32(t, name, shape):
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous CUDA fp32 tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


_ws_cache: dict = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    """Per-device scratch (single-stream use; pass `workspace=` for concurrent streams)."""
    key = torch.device(device).index
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def lora_linear_fwd_workspace_bytes(d: lora_dims) -> int:
    return int(lib.lora_linear_fwd_workspace_bytes(ctypes.byref(d)))


def lora_linear_bwd_workspace_bytes(d: lora_dims) -> int:
    return int(lib.lora_linear_bwd_workspace_bytes(ctypes.byref(d)))


def lora_last_launch_count() -> int:
    return int(lib.lora_last_launch_count())


def lora_captured_sync_words_free() -> int:
    """Free words of the sync-pool region used by calls made during graph capture."""
    return int(lib.lora_captured_sync_words_free())


def lora_profile_next_bwd(k2_begin=None, k2_end=None, k3_begin=None, k3_end=None) -> None:
    """Record torch.cuda.Events around the dX kernel and the dA / dB kernel of the
    next backward call on this thread (include/lora.h; one-shot)."""
    arr = (_vp * 4)(*[ev.cuda_event if ev is not None else None for ev in (k2_begin, k2_end, k3_begin, k3_end)])
    _check(lib.lora_profile_next_bwd(arr), "lora_profile_next_bwd")


def lora_device_check() -> None:
    _check(lib.lora_device_check(), "lora_device_check")


def _dropout(dropout):
    """(p, seed, offset[, keep_bits[, masked_x[, row_offset[, col_offset]]]]) -> lora_dropout
    (LoRA dropout; include/lora.h).  keep_bits: optional int32 device
    tensor [T, ceil(n/32)], masked_x: optional bf16 device tensor [T, n]; the forward
    fills them (keep mask, M . x) and the backward reads them instead of redrawing.
    row_offset / col_offset: this input's position in the full adapter input (its
    element (t, k) draws the mask of (t + row_offset, k + col_offset))."""
    p, seed, offset = dropout[:3]
    kb = dropout[3] if len(dropout) > 3 else None
    mx = dropout[4] if len(dropout) > 4 else None
    r0 = int(dropout[5]) if len(dropout) > 5 else 0
    c0 = int(dropout[6]) if len(dropout) > 6 else 0
    if kb is not None and (kb.dtype != torch.int32 or not kb.is_contiguous() or not kb.is_cuda):
        raise ValueError("keep_bits must be a contiguous int32 CUDA tensor [T, ceil(n/32)]")
    if mx is not None and (mx.dtype != torch.bfloat16 or not mx.is_contiguous() or not mx.is_cuda):
        raise ValueError("masked_x must be a contiguous bf16 CUDA tensor [T, n]")
    return lora_dropout(float(p), int(seed) & (2**64 - 1), int(offset) & (2**64 - 1),
                        kb.data_ptr() if kb is not None else None, mx.data_ptr() if mx is not None else None,
                        r0, c0)


def dropout_keep_bits(T, n, device="cuda"):
    """A keep-mask buffer for lora_dropout.keep_bits: int32 [T, ceil(n/32)]."""
    return torch.empty((T, (n + 31) // 32), dtype=torch.int32, device=device)


def lora_dropout_mask(T, n, dropout, device="cuda", stream=None):
    """Keep mask M [T, n] uint8 of lora_linear_{fwd,bwd}(..., dropout=(p, seed, offset))."""
    mask = torch.empty((T, n), dtype=torch.uint8, device=device)
    dr = _dropout(dropout)
    _check(lib.lora_dropout_mask(int(T), int(n), ctypes.byref(dr), _ptr(mask), _stream(stream)),
           "lora_dropout_mask")
    return mask


def lora_linear_fwd(x, w0, a, b, alpha, bias=None, y=None, h_out=None, want_h=True,
                    workspace=None, stream=None, dropout=None):
    """Forward of Eq. 1.  x [T,n], w0 [m,n], a [r,n], b [m,r]
    (bf16, CUDA).  dropout = (p, seed, offset) applies LoRA dropout to the
    adapter input.  Returns (y [T,m] bf16, h [T,r] fp32 or None)."""
    T, n = x.shape
    m, r = b.shape
    _bf16(x, "x", (T, n)); _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
    if bias is not None:
        _bf16(bias, "bias", (m,))
    if y is None:
        y = torch.empty((T, m), dtype=torch.bfloat16, device=x.device)
    _bf16(y, "y", (T, m))
    if h_out is None and want_h:
        h_out = torch.empty((T, r), dtype=torch.float32, device=x.device)
    if h_out is not None:
        _f32(h_out, "h_out", (T, r))
    d = dims(T, n, m, r, alpha)
    if dropout is not None:
        need = int(lib.lora_linear_fwd_dropout_workspace_bytes(ctypes.byref(d)))
        ws = workspace if workspace is not None else _workspace(need, x.device)
        dr = _dropout(dropout)
        st = lib.lora_linear_fwd_dropout(ctypes.byref(d), ctypes.byref(dr), _ptr(x), _ptr(w0), _ptr(a), _ptr(b),
                                         _ptr(bias), _ptr(y), _ptr(h_out), _ptr(ws), ws.numel(), _stream(stream))
        _check(st, "lora_linear_fwd_dropout")
        return y, h_out
    need = lora_linear_fwd_workspace_bytes(d)
    ws = workspace if workspace is not None else _workspace(need, x.device)
    st = lib.lora_linear_fwd(ctypes.byref(d), _ptr(x), _ptr(w0), _ptr(a), _ptr(b), _ptr(bias),
                             _ptr(y), _ptr(h_out), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "lora_linear_fwd")
    return y, h_out


def lora_linear_bwd(x, w0, a, b, dy, alpha, h_saved=None, want_dx=True, dx=None, da=None, db=None,
                    accumulate=False, want_da=True, want_db=True, workspace=None, stream=None, dropout=None):
    """Backward of Eq. 1; dropout as in lora_linear_fwd (same
    (p, seed, offset) as the forward).  Returns (dx [T,n] bf16 | None,
    dA [r,n] fp32 | None, dB [m,r] fp32 | None)."""
    T, n = x.shape
    m, r = b.shape
    _bf16(x, "x", (T, n)); _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
    _bf16(dy, "dy", (T, m))
    if h_saved is not None:
        _f32(h_saved, "h_saved", (T, r))
    if dx is None and want_dx:
        dx = torch.empty((T, n), dtype=torch.bfloat16, device=x.device)
    if dx is not None:
        _bf16(dx, "dx", (T, n))
    if da is None and want_da:
        da = torch.zeros((r, n), dtype=torch.float32, device=x.device)
    if db is None and want_db:
        db = torch.zeros((m, r), dtype=torch.float32, device=x.device)
    if da is not None:
        _f32(da, "da", (r, n))
    if db is not None:
        _f32(db, "db", (m, r))
    d = dims(T, n, m, r, alpha)
    if dropout is not None:
        need = int(lib.lora_linear_bwd_dropout_workspace_bytes(ctypes.byref(d)))
        ws = workspace if workspace is not None else _workspace(need, x.device)
        dr = _dropout(dropout)
        st = lib.lora_linear_bwd_dropout(ctypes.byref(d), ctypes.byref(dr), _ptr(x), _ptr(w0), _ptr(a), _ptr(b),
                                         _ptr(h_saved), _ptr(dy), _ptr(dx), _ptr(da), _ptr(db),
                                         1 if accumulate else 0, _ptr(ws), ws.numel(), _stream(stream))
        _check(st, "lora_linear_bwd_dropout")
        return dx, da, db
    need = lora_linear_bwd_workspace_bytes(d)
    ws = workspace if workspace is not None else _workspace(need, x.device)
    st = lib.lora_linear_bwd(ctypes.byref(d), _ptr(x), _ptr(w0), _ptr(a), _ptr(b), _ptr(h_saved),
                             _ptr(dy), _ptr(dx), _ptr(da), _ptr(db), 1 if accumulate else 0,
                             _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "lora_linear_bwd")
    return dx, da, db


def lora_merge(w0, a, b, alpha, w_out=None, stream=None):
    """W' = bf16(W0 + s B A) (Eq. 1 line 2).  w_out=w0 merges in place."""
    m, n = w0.shape
    r = a.shape[0]
    _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
    if w_out is None:
        w_out = torch.empty_like(w0)
    _bf16(w_out, "w_out", (m, n))
    d = dims(0, n, m, r, alpha)
    st = lib.lora_merge(ctypes.byref(d), _ptr(w0), _ptr(a), _ptr(b), _ptr(w_out), _stream(stream))
    _check(st, "lora_merge")
    return w_out


def lora_linear_fwd_grouped(problems, alphas, outs=None, workspace=None, stream=None, dropouts=None):
    """Grouped forward (one persistent launch for the fused GEMMs).

    problems: list of (x, w0, a, b, bias_or_None); alphas: list of floats;
    outs: optional list of (y, h_out).  Returns the list of (y, h)."""
    G = len(problems)
    if not 1 <= G <= LORA_MAX_GROUP:
        raise ValueError(f"1 <= len(problems) <= {LORA_MAX_GROUP}")
    dims_arr = (lora_dims * G)()
    probs = (lora_fwd_problem * G)()
    res = []
    for g, (x, w0, a, b, bias) in enumerate(problems):
        T, n = x.shape
        m, r = b.shape
        _bf16(x, "x", (T, n)); _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
        y, h = outs[g] if outs is not None else (None, None)
        if y is None:
            y = torch.empty((T, m), dtype=torch.bfloat16, device=x.device)
        if h is None:
            h = torch.empty((T, r), dtype=torch.float32, device=x.device)
        dims_arr[g] = dims(T, n, m, r, alphas[g])
        probs[g] = lora_fwd_problem(_ptr(x), _ptr(w0), _ptr(a), _ptr(b), _ptr(bias), _ptr(y), _ptr(h))
        res.append((y, h))
    if dropouts is not None:   # one (p, seed, offset) per problem
        drs = (lora_dropout * G)(*[_dropout(dr) for dr in dropouts])
        need = int(lib.lora_linear_fwd_grouped_dropout_workspace_bytes(G, dims_arr))
        ws = workspace if workspace is not None else _workspace(need, problems[0][0].device)
        _check(lib.lora_linear_fwd_grouped_dropout(G, dims_arr, drs, probs, _ptr(ws), ws.numel(), _stream(stream)),
               "lora_linear_fwd_grouped_dropout")
        return res
    need = int(lib.lora_linear_fwd_grouped_workspace_bytes(G, dims_arr))
    ws = workspace if workspace is not None else _workspace(need, problems[0][0].device)
    _check(lib.lora_linear_fwd_grouped(G, dims_arr, probs, _ptr(ws), ws.numel(), _stream(stream)),
           "lora_linear_fwd_grouped")
    return res


def lora_linear_bwd_grouped(problems, alphas, outs=None, accumulate=False, workspace=None, stream=None,
                            want_dx=True, want_da=True, want_db=True, dropouts=None):
    """Grouped backward.  problems: list of (x, w0, a, b, dy, h_saved_or_None);
    outs: optional list of (dx, da, db); want_*=False passes NULL for that output
    of every problem (not allocated).  Returns the list of (dx, da, db)."""
    G = len(problems)
    if not 1 <= G <= LORA_MAX_GROUP:
        raise ValueError(f"1 <= len(problems) <= {LORA_MAX_GROUP}")
    dims_arr = (lora_dims * G)()
    probs = (lora_bwd_problem * G)()
    res = []
    for g, (x, w0, a, b, dy, h) in enumerate(problems):
        T, n = x.shape
        m, r = b.shape
        _bf16(x, "x", (T, n)); _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
        _bf16(dy, "dy", (T, m))
        dx, da, db = outs[g] if outs is not None else (None, None, None)
        if dx is None and want_dx:
            dx = torch.empty((T, n), dtype=torch.bfloat16, device=x.device)
        if da is None and want_da:
            da = torch.zeros((r, n), dtype=torch.float32, device=x.device)
        if db is None and want_db:
            db = torch.zeros((m, r), dtype=torch.float32, device=x.device)
        dx, da, db = (dx if want_dx else None), (da if want_da else None), (db if want_db else None)
        dims_arr[g] = dims(T, n, m, r, alphas[g])
        probs[g] = lora_bwd_problem(_ptr(x), _ptr(w0), _ptr(a), _ptr(b), _ptr(h), _ptr(dy), _ptr(dx), _ptr(da),
                                    _ptr(db))
        res.append((dx, da, db))
    if dropouts is not None:
        drs = (lora_dropout * G)(*[_dropout(dr) for dr in dropouts])
        need = int(lib.lora_linear_bwd_grouped_dropout_workspace_bytes(G, dims_arr))
        ws = workspace if workspace is not None else _workspace(need, problems[0][0].device)
        _check(lib.lora_linear_bwd_grouped_dropout(G, dims_arr, drs, probs, 1 if accumulate else 0, _ptr(ws),
                                                   ws.numel(), _stream(stream)), "lora_linear_bwd_grouped_dropout")
        return res
    need = int(lib.lora_linear_bwd_grouped_workspace_bytes(G, dims_arr))
    ws = workspace if workspace is not None else _workspace(need, problems[0][0].device)
    _check(lib.lora_linear_bwd_grouped(G, dims_arr, probs, 1 if accumulate else 0, _ptr(ws), ws.numel(),
                                       _stream(stream)), "lora_linear_bwd_grouped")
    return res


def lora_adam_step(tensors, step, lr, betas=(0.9, 0.999), eps=1e-8, stream=None):
    """One bias-corrected Adam step for adapter tensors in ONE launch (SURVEY.md
    8(f) N3; include/lora.h).  tensors: list of (param bf16, grad fp32, m fp32,
    v fp32, master fp32 or None), all CUDA, same numel per entry; updated in place."""
    n = len(tensors)
    if not 1 <= n <= LORA_ADAM_MAX_TENSORS:
        raise ValueError(f"1 <= len(tensors) <= {LORA_ADAM_MAX_TENSORS}")
    arr = (lora_adam_tensor * n)()
    for i, (p, g, m, v, w) in enumerate(tensors):
        numel = p.numel()
        if p.dtype != torch.bfloat16 or any(t.dtype != torch.float32 or t.numel() != numel
                                            for t in (g, m, v) + ((w,) if w is not None else ())):
            raise ValueError(f"tensor {i}: param bf16 and grad/m/v/master fp32 of equal numel")
        for t in (p, g, m, v) + ((w,) if w is not None else ()):
            if not t.is_contiguous() or not t.is_cuda:
                raise ValueError(f"tensor {i}: contiguous CUDA tensors required")
        arr[i] = lora_adam_tensor(_ptr(p), _ptr(w), _ptr(g), _ptr(m), _ptr(v), numel)
    hp = lora_adam_hparams(float(lr), float(betas[0]), float(betas[1]), float(eps))
    _check(lib.lora_adam_step(n, arr, ctypes.byref(hp), int(step), _stream(stream)), "lora_adam_step")


# ------------------------------------------------ merged-weight export (N3)
def _dt_code(dtype):
    if dtype in (torch.float32, "float32", "f32"):
        return 0
    if dtype in (torch.bfloat16, "bfloat16", "bf16"):
        return 1
    raise ValueError(f"unsupported dtype {dtype} (float32 / bfloat16)")


def write_safetensors(path, tensors):
    """lora_write_safetensors: {name: contiguous CPU torch tensor (float32 / bfloat16)}."""
    items = list(tensors.items())
    arr = (lora_host_tensor * max(1, len(items)))()
    keep = []
    for i, (name, t) in enumerate(items):
        t = t.contiguous()
        keep.append(t)
        shp = (ctypes.c_int64 * 4)(*(list(t.shape) + [0] * (4 - t.dim())))
        arr[i] = lora_host_tensor(name.encode(), _dt_code(t.dtype), t.dim(), shp, t.data_ptr())
    _check(lib.lora_write_safetensors(str(path).encode(), len(items), arr), "lora_write_safetensors")


def export_merged(path, entries, stream=None):
    """lora_export_merged.  entries: list of (name, w0, a, b, alpha) -- merged on the
    GPU into W0 + s B A -- or (name, tensor) -- written as it is (CUDA tensors)."""
    arr = (lora_export_tensor * max(1, len(entries)))()
    for i, ent in enumerate(entries):
        name = ent[0].encode()
        if len(ent) == 5:
            _, w0, a, b, alpha = ent
            m, n = w0.shape
            r = a.shape[0]
            _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
            arr[i] = lora_export_tensor(name, _ptr(w0), _ptr(a), _ptr(b), dims(0, n, m, r, alpha), 1, 2,
                                        (ctypes.c_int64 * 4)(m, n, 0, 0))
        else:
            t = ent[1]
            if not (t.is_cuda and t.is_contiguous()):
                raise ValueError(f"{ent[0]}: must be a contiguous CUDA tensor")
            shp = (ctypes.c_int64 * 4)(*(list(t.shape) + [0] * (4 - t.dim())))
            arr[i] = lora_export_tensor(name, _ptr(t), None, None, lora_dims(0, 0, 0, 0, 0.0), _dt_code(t.dtype),
                                        t.dim(), shp)
    _check(lib.lora_export_merged(str(path).encode(), len(entries), arr, _stream(stream)), "lora_export_merged")


# ------------------------------------------------ decoder-layer pieces (N4)
def lora_rmsnorm_fwd(x, g, eps, res=None, y=None, x2_out=None, rstd=None, stream=None):
    """y = g * (x2 * rstd), x2 = x (+ res).  Returns (y, rstd [T] fp32)."""
    T, d = x.shape
    _bf16(x, "x", (T, d)); _bf16(g, "g", (d,))
    if res is not None:
        _bf16(res, "res", (T, d))
    y = torch.empty_like(x) if y is None else y
    rstd = torch.empty(T, dtype=torch.float32, device=x.device) if rstd is None else rstd
    _check(lib.lora_rmsnorm_fwd(T, d, float(eps), _ptr(x), _ptr(res), _ptr(g), _ptr(y), _ptr(x2_out), _ptr(rstd),
                                _stream(stream)), "lora_rmsnorm_fwd")
    return y, rstd


def lora_rmsnorm_bwd(dy, x2, g, rstd, dres=None, dx=None, stream=None):
    T, d = dy.shape
    dx = torch.empty_like(dy) if dx is None else dx
    _check(lib.lora_rmsnorm_bwd(T, d, _ptr(dy), _ptr(x2), _ptr(g), _ptr(rstd), _ptr(dres), _ptr(dx),
                                _stream(stream)), "lora_rmsnorm_bwd")
    return dx


def lora_rope(q, heads, head_dim, theta=10000.0, pos0=0, inverse=False, stream=None):
    """In place on q [T, >= heads * head_dim] (row stride q.stride(0))."""
    T = q.shape[0]
    _check(lib.lora_rope(T, int(heads), int(head_dim), q.stride(0), int(pos0), float(theta), 1 if inverse else 0,
                         _ptr(q), _stream(stream)), "lora_rope")
    return q


def lora_swiglu_fwd(gate, up, out=None, stream=None):
    out = torch.empty_like(gate) if out is None else out
    _check(lib.lora_swiglu_fwd(gate.numel(), _ptr(gate), _ptr(up), _ptr(out), _stream(stream)), "lora_swiglu_fwd")
    return out


def lora_swiglu_bwd(gate, up, da, dgate=None, dup=None, stream=None):
    dgate = torch.empty_like(gate) if dgate is None else dgate
    dup = torch.empty_like(up) if dup is None else dup
    _check(lib.lora_swiglu_bwd(gate.numel(), _ptr(gate), _ptr(up), _ptr(da), _ptr(dgate), _ptr(dup),
                               _stream(stream)), "lora_swiglu_bwd")
    return dgate, dup


def lora_sum_bf16(srcs, dst=None, stream=None):
    dst = torch.empty_like(srcs[0]) if dst is None else dst
    arr = (_vp * len(srcs))(*[_ptr(t) for t in srcs])
    _check(lib.lora_sum_bf16(srcs[0].numel(), len(srcs), arr, _ptr(dst), _stream(stream)), "lora_sum_bf16")
    return dst

"""Tensor parallelism for the LoRA linear, one process per GPU.

PAPER.md:122: "JORA parallelizes all parameters of the Llama model using JAX's
positional sharding module ... Projection and Embedding layers are sharded on
the non-sequential dimension."  Read (R10-R13) as Megatron column /
row parallelism inside the decoder block:

  COLUMN (q, k, v, gate, up): W0 [m, n] and B [m, r] split on m (d_out),
      A [r, n] replicated.  fwd: local, no collective.  bwd: dX and dA are
      partial sums -> all-reduce; dB local.
  ROW (o, down): W0 and A split on n (d_in), B replicated.  fwd: y is a
      partial sum -> all-reduce (bias added once); bwd: dB partial ->
      all-reduce; dX, dA local.

Partial sums are reduced with a SUM (no 1/N; R12).  The collectives run in
liblora.so over NCCL (lora_comm_*); torch.distributed is used only to
broadcast the NCCL unique id (plumbing).  The sharding functions here are the
host logic; they are covered on CPU by tests/test_tp_gloo.py.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

COLUMN = 0
ROW = 1
MODES = {"column": COLUMN, "row": ROW}


@dataclass(frozen=True)
class ShardSpec:
    """How one LoRA linear is split across `world` ranks."""
    mode: int          # COLUMN or ROW
    world: int
    rank: int
    n: int             # full d_in
    m: int             # full d_out

    def __post_init__(self):
        if self.world < 1 or not (0 <= self.rank < self.world):
            raise ValueError(f"bad rank {self.rank} / world {self.world}")
        axis, extent = ("d_out", self.m) if self.mode == COLUMN else ("d_in", self.n)
        if extent % self.world != 0:
            raise ValueError(f"divisibility violation: {axis} = {extent} is not divisible by N = {self.world}")
        if (extent // self.world) % 8 != 0:
            raise ValueError(f"shard of {axis} = {extent // self.world} is not a multiple of 8 (TMA rows)")

    @property
    def local_n(self) -> int:
        return self.n // self.world if self.mode == ROW else self.n

    @property
    def local_m(self) -> int:
        return self.m // self.world if self.mode == COLUMN else self.m

    def slice(self):
        """Slice of the sharded axis owned by this rank."""
        ext = self.local_m if self.mode == COLUMN else self.local_n
        return slice(self.rank * ext, (self.rank + 1) * ext)


def shard_params(spec: ShardSpec, w0, a, b, bias=None):
    """Local (W0, A, B, bias) of this rank (works on numpy arrays and torch tensors).
    COLUMN: W0[rows], B[rows], A full, bias[rows].  ROW: W0[:, cols], A[:, cols],
    B full, bias full (added once by rank 0)."""
    sl = spec.slice()
    if spec.mode == COLUMN:
        return w0[sl], a, b[sl], (bias[sl] if bias is not None else None)
    return w0[:, sl], a[:, sl], b, bias


def shard_input(spec: ShardSpec, x):
    """Local activation: COLUMN takes the full x; ROW takes x[:, cols]."""
    return x if spec.mode == COLUMN else x[:, spec.slice()]


def shard_output_grad(spec: ShardSpec, dy):
    """Local upstream gradient: COLUMN takes dY[:, rows]; ROW the full dY."""
    return dy[:, spec.slice()] if spec.mode == COLUMN else dy


def partial_outputs(spec: ShardSpec):
    """Which results are partial sums on each rank (reduced by a SUM)."""
    if spec.mode == COLUMN:
        return {"y": False, "dx": True, "da": True, "db": False}
    return {"y": True, "dx": False, "da": False, "db": True}


# --------------------------------------------------------------------- runtime
class LoraComm:
    """An NCCL communicator owned by liblora.so (lora_comm_*), created from a
    unique id broadcast over an existing torch.distributed process group."""

    def __init__(self, group=None):
        import os

        import torch
        import torch.distributed as dist

        from . import build as _build
        from . import lib, _check
        nccl = _build.nccl_library()
        if nccl and "LORA_NCCL_LIB" not in os.environ:
            os.environ["LORA_NCCL_LIB"] = nccl
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(lib.lora_comm_unique_id(uid), "lora_comm_unique_id")
        if self.world > 1:
            t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0, group=group)
            uid = ctypes.create_string_buffer(bytes(t.cpu().tolist()), 128)
        self._h = ctypes.c_void_p()
        _check(lib.lora_comm_init(self.world, self.rank, uid, ctypes.byref(self._h)), "lora_comm_init")

    @property
    def handle(self):
        return self._h

    def allreduce(self, t, stream=None):
        import torch

        from . import lib, _check, _stream
        dt = 0 if t.dtype == torch.float32 else 1
        _check(lib.lora_allreduce(self._h, t.data_ptr(), t.numel(), dt, _stream(stream)), "lora_allreduce")

    def close(self):
        from . import lib
        if self._h:
            lib.lora_comm_destroy(self._h)
            self._h = ctypes.c_void_p()


def tp_linear_fwd(comm: LoraComm, spec: ShardSpec, x, w0, a, b, alpha, bias=None, y=None, h_out=None,
                  workspace=None, stream=None, dropout=None):
    """lora_tp_linear_fwd on local shards.  Returns (y [T, local_m], h [T, r]).
    dropout: (p, seed, offset[, keep_bits[, masked_x]]) of the FULL input (keep_bits /
    masked_x local) -> lora_tp_linear_fwd_dropout (row mode draws its shard's columns)."""
    import torch

    from . import _bf16, _check, _dropout, _ptr, _stream, _workspace, dims, lib, lora_linear_fwd_workspace_bytes
    T = x.shape[0]
    r = a.shape[0]
    n, m = spec.local_n, spec.local_m
    _bf16(x, "x", (T, n)); _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
    if y is None:
        y = torch.empty((T, m), dtype=torch.bfloat16, device=x.device)
    if h_out is None:
        h_out = torch.empty((T, r), dtype=torch.float32, device=x.device)
    d = dims(T, n, m, r, alpha)
    if dropout is not None:
        dr = _dropout(dropout)
        need = int(lib.lora_linear_fwd_dropout_workspace_bytes(ctypes.byref(d)))
        ws = workspace if workspace is not None else _workspace(need, x.device)
        _check(lib.lora_tp_linear_fwd_dropout(comm.handle, spec.mode, ctypes.byref(d), ctypes.byref(dr), _ptr(x),
                                              _ptr(w0), _ptr(a), _ptr(b), _ptr(bias), _ptr(y), _ptr(h_out), _ptr(ws),
                                              ws.numel(), _stream(stream)), "lora_tp_linear_fwd_dropout")
        return y, h_out
    ws = workspace if workspace is not None else _workspace(lora_linear_fwd_workspace_bytes(d), x.device)
    _check(lib.lora_tp_linear_fwd(comm.handle, spec.mode, ctypes.byref(d), _ptr(x), _ptr(w0), _ptr(a), _ptr(b),
                                  _ptr(bias), _ptr(y), _ptr(h_out), _ptr(ws), ws.numel(), _stream(stream)),
           "lora_tp_linear_fwd")
    return y, h_out


def tp_linear_bwd(comm: LoraComm, spec: ShardSpec, x, w0, a, b, dy, alpha, h_saved=None, dx=None, da=None,
                  db=None, accumulate=False, reduce_lora_grads=True, want_dx=True, workspace=None, stream=None,
                  dropout=None):
    """lora_tp_linear_bwd on local shards.  Returns (dx, dA, dB) local tensors
    (dx / dA / dB already summed across ranks where they are partial).  dropout:
    as tp_linear_fwd (the same tuple as the forward) -> lora_tp_linear_bwd_dropout."""
    import torch

    from . import _check, _dropout, _ptr, _stream, _workspace, dims, lib
    T = x.shape[0]
    r = a.shape[0]
    n, m = spec.local_n, spec.local_m
    if dx is None and want_dx:
        dx = torch.empty((T, n), dtype=torch.bfloat16, device=x.device)
    if da is None:
        da = torch.zeros((r, n), dtype=torch.float32, device=x.device)
    if db is None:
        db = torch.zeros((m, r), dtype=torch.float32, device=x.device)
    d = dims(T, n, m, r, alpha)
    if dropout is not None:
        dr = _dropout(dropout)
        need = int(lib.lora_tp_linear_bwd_dropout_workspace_bytes(ctypes.byref(d)))
        ws = workspace if workspace is not None else _workspace(need, x.device)
        _check(lib.lora_tp_linear_bwd_dropout(comm.handle, spec.mode, ctypes.byref(d), ctypes.byref(dr), _ptr(x),
                                              _ptr(w0), _ptr(a), _ptr(b), _ptr(h_saved), _ptr(dy), _ptr(dx), _ptr(da),
                                              _ptr(db), 1 if accumulate else 0, 1 if reduce_lora_grads else 0,
                                              _ptr(ws), ws.numel(), _stream(stream)), "lora_tp_linear_bwd_dropout")
        return dx, da, db
    need = int(lib.lora_tp_linear_bwd_workspace_bytes(ctypes.byref(d)))
    ws = workspace if workspace is not None else _workspace(need, x.device)
    _check(lib.lora_tp_linear_bwd(comm.handle, spec.mode, ctypes.byref(d), _ptr(x), _ptr(w0), _ptr(a), _ptr(b),
                                  _ptr(h_saved), _ptr(dy), _ptr(dx), _ptr(da), _ptr(db), 1 if accumulate else 0,
                                  1 if reduce_lora_grads else 0, _ptr(ws), ws.numel(), _stream(stream)),
           "lora_tp_linear_bwd")
    return dx, da, db


def tp_linear_bwd_column_group(comm: LoraComm, specs, problems, alphas, dx_sum=None, want_dx=True, outs=None,
                               reduce_lora_grads=True, workspace=None, stream=None, dropouts=None):
    """lora_tp_linear_bwd_column_group: the backward of COLUMN-parallel linears that
    read the same input (q/k/v, gate/up).  problems: list of
    (x, w0, a, b, dy, h_saved) local shards with the SAME x tensor.  The members'
    dX partials are summed into dx_sum (the gradient w.r.t. the shared input) and
    all-reduced once.  dropouts: one (p, seed, offset[, keep_bits[, masked_x]]) per
    member (the forward's) -> lora_tp_linear_bwd_column_group_dropout.
    Returns (dx_sum, [(dx_g, dA_g, dB_g)])."""
    import torch

    from . import _check, _dropout, _ptr, _stream, _workspace, dims, lib, lora_bwd_problem, lora_dims, lora_dropout
    G = len(problems)
    x = problems[0][0]
    T = x.shape[0]
    n = specs[0].local_n
    if any(sp.mode != COLUMN for sp in specs):
        raise ValueError("tp_linear_bwd_column_group is for COLUMN-parallel linears")
    if any(p[0] is not x and p[0].data_ptr() != x.data_ptr() for p in problems):
        raise ValueError("all problems must share the same input tensor x")
    if dx_sum is None and want_dx:
        dx_sum = torch.empty((T, n), dtype=torch.bfloat16, device=x.device)
    dims_arr = (lora_dims * G)()
    probs = (lora_bwd_problem * G)()
    res = []
    for g, ((xg, w0, a, b, dy, h), sp) in enumerate(zip(problems, specs)):
        r = a.shape[0]
        m = sp.local_m
        dx, da, db = outs[g] if outs is not None else (None, None, None)
        if dx is None and want_dx:
            dx = torch.empty((T, n), dtype=torch.bfloat16, device=x.device)
        if da is None:
            da = torch.zeros((r, n), dtype=torch.float32, device=x.device)
        if db is None:
            db = torch.zeros((m, r), dtype=torch.float32, device=x.device)
        dims_arr[g] = dims(T, n, m, r, alphas[g])
        probs[g] = lora_bwd_problem(_ptr(xg), _ptr(w0), _ptr(a), _ptr(b), _ptr(h), _ptr(dy), _ptr(dx), _ptr(da),
                                    _ptr(db))
        res.append((dx, da, db))
    if dropouts is not None:
        drs = (lora_dropout * G)(*[_dropout(dr) for dr in dropouts])
        need = int(lib.lora_tp_linear_bwd_column_group_dropout_workspace_bytes(G, dims_arr))
        ws = workspace if workspace is not None else _workspace(need, x.device)
        _check(lib.lora_tp_linear_bwd_column_group_dropout(comm.handle, G, dims_arr, drs, probs, _ptr(dx_sum), 0,
                                                           1 if reduce_lora_grads else 0, _ptr(ws), ws.numel(),
                                                           _stream(stream)), "lora_tp_linear_bwd_column_group_dropout")
        return dx_sum, res
    need = int(lib.lora_tp_linear_bwd_column_group_workspace_bytes(G, dims_arr))
    ws = workspace if workspace is not None else _workspace(need, x.device)
    _check(lib.lora_tp_linear_bwd_column_group(comm.handle, G, dims_arr, probs, _ptr(dx_sum), 0,
                                               1 if reduce_lora_grads else 0, _ptr(ws), ws.numel(),
                                               _stream(stream)), "lora_tp_linear_bwd_column_group")
    return dx_sum, res


# ------------------------------------------------- comm-fused epilogues (N2)
class _DevView:
    """__cuda_array_interface__ over raw device memory (a view into a lora_symm)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class SymmBuffer:
    """A symmetric device buffer of liblora.so (lora_symm_*):
    the same size on every rank, peers mapped with CUDA IPC.  The fused TP calls
    write their partial outputs and results into regions of it (byte offsets).

    SymmBuffer(nbytes, group) -- one per rank of a torch.distributed group
        (IPC handles all-gathered over it).
    SymmBuffer.local_group(nranks, nbytes) -- N buffers of THIS process on the
        current device, joined as N virtual ranks (runs the protocol on one GPU)."""

    def __init__(self, nbytes: int, group=None, _connect=True):
        import torch.distributed as dist

        from . import _check, lib
        self._h = ctypes.c_void_p()
        _check(lib.lora_symm_create(int(nbytes), ctypes.byref(self._h)), "lora_symm_create")
        self.nbytes = int(lib.lora_symm_bytes(self._h))
        self.world, self.rank = 1, 0
        if not _connect:
            return
        if dist.is_initialized():
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        mine = ctypes.create_string_buffer(64)
        _check(lib.lora_symm_ipc_handle(self._h, mine), "lora_symm_ipc_handle")
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, bytes(mine.raw), group=group)
        else:
            handles = [bytes(mine.raw)]
        blob = ctypes.create_string_buffer(b"".join(handles), 64 * self.world)
        _check(lib.lora_symm_connect(self._h, self.world, self.rank, blob), "lora_symm_connect")

    @classmethod
    def local_group(cls, nranks: int, nbytes: int):
        from . import _check, lib
        bufs = [cls(nbytes, _connect=False) for _ in range(nranks)]
        arr = (ctypes.c_void_p * nranks)(*[b._h.value for b in bufs])
        _check(lib.lora_symm_connect_local(nranks, arr), "lora_symm_connect_local")
        for r, b in enumerate(bufs):
            b.world, b.rank = nranks, r
        return bufs

    @property
    def handle(self):
        return self._h

    @property
    def last_placement(self):
        """1 co-resident reducer, 2 reducer after the GEMM, 3 virtual ranks (split SMs)."""
        from . import lib
        return {0: None, 1: "coresident", 2: "after_gemm", 3: "split_sms"}[lib.lora_symm_last_placement(self._h)]

    def view(self, offset: int, shape, dtype="bf16"):
        """A torch tensor over [offset, ...) of this rank's data region."""
        import torch

        from . import lib
        base = lib.lora_symm_ptr(self._h)
        typestr = {"bf16": "<f2", "f32": "<f4"}[dtype]
        t = torch.as_tensor(_DevView(base + int(offset), shape, typestr), device="cuda")
        return t.view(torch.bfloat16) if dtype == "bf16" else t

    def close(self):
        from . import lib
        if self._h:
            lib.lora_symm_destroy(self._h)
            self._h = ctypes.c_void_p()


def tp_linear_fwd_fused(symm: SymmBuffer, spec: ShardSpec, x, w0, a, b, alpha, bias=None, part_offset=0,
                        y_offset=None, h_out=None, workspace=None, stream=None):
    """lora_tp_linear_fwd_fused: ROW-parallel forward with the y all-reduce fused
    into the GEMM.  Returns (y [T, m] -- a view of the symmetric buffer, valid until
    the next fused call writing that region --, h [T, r])."""
    import torch

    from . import _bf16, _check, _ptr, _stream, _workspace, dims, lib, lora_linear_fwd_workspace_bytes
    if spec.mode != ROW:
        raise ValueError("tp_linear_fwd_fused is the ROW-parallel forward (its y is a partial sum)")
    T, r = x.shape[0], a.shape[0]
    n, m = spec.local_n, spec.local_m
    _bf16(x, "x", (T, n)); _bf16(w0, "w0", (m, n)); _bf16(a, "a", (r, n)); _bf16(b, "b", (m, r))
    yb = T * m * 2
    if y_offset is None:
        y_offset = part_offset + (yb + 255) // 256 * 256
    if h_out is None:
        h_out = torch.empty((T, r), dtype=torch.float32, device=x.device)
    d = dims(T, n, m, r, alpha)
    ws = workspace if workspace is not None else _workspace(lora_linear_fwd_workspace_bytes(d), x.device)
    _check(lib.lora_tp_linear_fwd_fused(symm.handle, ctypes.byref(d), _ptr(x), _ptr(w0), _ptr(a), _ptr(b),
                                        _ptr(bias), int(part_offset), int(y_offset), _ptr(h_out), _ptr(ws),
                                        ws.numel(), _stream(stream)), "lora_tp_linear_fwd_fused")
    return symm.view(y_offset, (T, m)), h_out


def tp_linear_bwd_column_group_fused(symm: SymmBuffer, specs, problems, alphas, comm=None, part_offset=0,
                                     dx_offset=None, outs=None, reduce_lora_grads=False, workspace=None,
                                     stream=None):
    """lora_tp_linear_bwd_column_group_fused: the COLUMN group backward with the dX
    all-reduce (over ranks and members) fused into the grouped dX GEMM.
    problems: (x, w0, a, b, dy, h_saved) local shards sharing x.  Returns
    (dx_sum [T, n] -- a view of the symmetric buffer --, [(dA_g, dB_g)])."""
    import torch

    from . import _check, _ptr, _stream, _workspace, dims, lib, lora_bwd_problem, lora_dims
    G = len(problems)
    x = problems[0][0]
    T, n = x.shape[0], specs[0].local_n
    if any(sp.mode != COLUMN for sp in specs):
        raise ValueError("the fused column-group backward is for COLUMN-parallel linears")
    xb = T * n * 2
    if dx_offset is None:
        dx_offset = part_offset + (G * xb + 255) // 256 * 256
    dims_arr = (lora_dims * G)()
    probs = (lora_bwd_problem * G)()
    res = []
    for g, ((xg, w0, a, b, dy, h), sp) in enumerate(zip(problems, specs)):
        r, m = a.shape[0], sp.local_m
        da, db = outs[g] if outs is not None else (None, None)
        if da is None:
            da = torch.empty((r, n), dtype=torch.float32, device=x.device)
        if db is None:
            db = torch.empty((m, r), dtype=torch.float32, device=x.device)
        dims_arr[g] = dims(T, n, m, r, alphas[g])
        probs[g] = lora_bwd_problem(_ptr(xg), _ptr(w0), _ptr(a), _ptr(b), _ptr(h), _ptr(dy), None, _ptr(da),
                                    _ptr(db))
        res.append((da, db))
    need = int(lib.lora_linear_bwd_grouped_workspace_bytes(G, dims_arr))
    ws = workspace if workspace is not None else _workspace(need, x.device)
    _check(lib.lora_tp_linear_bwd_column_group_fused(symm.handle, comm.handle if comm is not None else None, G,
                                                     dims_arr, probs, int(part_offset), int(dx_offset),
                                                     1 if reduce_lora_grads else 0, _ptr(ws), ws.numel(),
                                                     _stream(stream)), "lora_tp_linear_bwd_column_group_fused")
    return symm.view(dx_offset, (T, n)), res

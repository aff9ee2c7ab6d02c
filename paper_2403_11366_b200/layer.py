"""One Llama-2 decoder layer with LoRA on all seven projections -- the second
workload of SURVEY.md 8(f) N4 ("full Llama-2 decoder-layer train step at seq 4096
under TP: attention, RMSNorm, RoPE, SwiGLU"; PAPER.md:90 -- JORA builds on a
Llama-2 implementation -- and :195, the long single-sequence RAFT setting).

Composition only: every step runs in liblora.so (the fused LoRA linears, grouped
where projections share an input; RMSNorm, RoPE, SwiGLU and the residual sums)
except the attention, which is the cuDNN SDPA library call (like cuBLAS for a
plain GEMM).  W0 and the norm weights are frozen (PAPER.md:111,
:113): the backward yields dx and dA / dB of the seven adapters.

Tensor parallelism (R10-R12) with a LoraComm: q/k/v and
gate/up are COLUMN-parallel groups (heads and the FFN split over ranks; their dX
w.r.t. the shared input is summed and all-reduced once per group), o and down
are ROW-parallel (their y all-reduced).  The oracle is oracle/layer.py.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from . import (lora_linear_bwd, lora_linear_bwd_grouped, lora_linear_fwd, lora_linear_fwd_grouped, lora_rmsnorm_bwd,
               lora_rmsnorm_fwd, lora_rope, lora_sum_bf16, lora_swiglu_bwd, lora_swiglu_fwd)
from . import tp as _tp

COLUMN_GROUPS = (("q", "k", "v"), ("gate", "up"))
ROW = ("o", "down")
PROJ = ("q", "k", "v", "o", "gate", "up", "down")


def _sdpa(q, k, v):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION]):
        return F.scaled_dot_product_attention(q, k, v, is_causal=True)


class LlamaLayerLoRA:
    """params: device bf16 tensors w0_<p> [m, n], a_<p> [r, n], b_<p> [m, r] for the
    seven projections (LOCAL shards under TP) and the RMSNorm weights g1, g2 [d];
    cfg: heads (global), head_dim, eps, theta, alpha.  comm: a tp.LoraComm or None."""

    def __init__(self, params, cfg, comm=None):
        self.P, self.cfg, self.comm = params, cfg, comm
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.heads = cfg["heads"] // self.world
        self.D = cfg["head_dim"]
        self.d = params["g1"].shape[0]
        self.alpha = cfg["alpha"]
        self.ctx = None
        if comm is not None:
            d, F_ = self.d, cfg["ffn"]
            self.specs = {p: _tp.ShardSpec(_tp.COLUMN, self.world, self.rank, d, d) for p in ("q", "k", "v")}
            self.specs.update({p: _tp.ShardSpec(_tp.COLUMN, self.world, self.rank, d, F_) for p in ("gate", "up")})
            self.specs["o"] = _tp.ShardSpec(_tp.ROW, self.world, self.rank, d, d)
            self.specs["down"] = _tp.ShardSpec(_tp.ROW, self.world, self.rank, F_, d)

    def _w(self, p):
        return self.P["w0_" + p], self.P["a_" + p], self.P["b_" + p]

    # ------------------------------------------------------------------ forward
    def forward(self, x, stream=None):
        P, c = self.P, self.cfg
        T = x.shape[0]
        h1, rstd1 = lora_rmsnorm_fwd(x, P["g1"], c["eps"], stream=stream)
        qkv = lora_linear_fwd_grouped([(h1, *self._w(p), None) for p in ("q", "k", "v")], [self.alpha] * 3,
                                      stream=stream)
        (q, hq), (k, hk), (v, hv) = qkv
        lora_rope(q, self.heads, self.D, c["theta"], stream=stream)
        lora_rope(k, self.heads, self.D, c["theta"], stream=stream)
        qd, kd, vd = (t.view(T, self.heads, self.D).transpose(0, 1).unsqueeze(0).detach().requires_grad_(True)
                      for t in (q, k, v))
        with torch.enable_grad():
            att4 = _sdpa(qd, kd, vd)                                   # [1, H, T, D]
        attn = att4.detach()[0].transpose(0, 1).reshape(T, self.heads * self.D).contiguous()
        o, ho = self._row_fwd("o", attn, stream)
        x2 = torch.empty_like(x)
        h2, rstd2 = lora_rmsnorm_fwd(x, P["g2"], c["eps"], res=o, x2_out=x2, stream=stream)
        (g, hg), (u, hu) = lora_linear_fwd_grouped([(h2, *self._w(p), None) for p in ("gate", "up")],
                                                   [self.alpha] * 2, stream=stream)
        a = lora_swiglu_fwd(g, u, stream=stream)
        dn, hdn = self._row_fwd("down", a, stream)
        out = lora_sum_bf16([x2, dn], stream=stream)
        self.ctx = dict(x=x, h1=h1, rstd1=rstd1, hq=hq, hk=hk, hv=hv, qd=qd, kd=kd, vd=vd, att4=att4, attn=attn,
                        ho=ho, x2=x2, h2=h2, rstd2=rstd2, g=g, u=u, hg=hg, hu=hu, a=a, hdn=hdn)
        return out

    def _row_fwd(self, p, inp, stream):
        if self.comm is None:
            return lora_linear_fwd(inp, *self._w(p), self.alpha, stream=stream)
        return _tp.tp_linear_fwd(self.comm, self.specs[p], inp, *self._w(p), self.alpha, stream=stream)

    def _row_bwd(self, p, inp, dy, h, stream):
        if self.comm is None:
            return lora_linear_bwd(inp, *self._w(p), dy, self.alpha, h_saved=h, stream=stream)
        return _tp.tp_linear_bwd(self.comm, self.specs[p], inp, *self._w(p), dy, self.alpha, h_saved=h,
                                 stream=stream)

    def _col_group_bwd(self, names, inp, dys, hs, stream):
        """Backward of a column group sharing `inp`: (dX w.r.t. inp summed over members
        -- and, under TP, all-reduced --, [(dA, dB)])."""
        probs = [(inp, *self._w(p), dy, h) for p, dy, h in zip(names, dys, hs)]
        if self.comm is None:
            res = lora_linear_bwd_grouped(probs, [self.alpha] * len(names), stream=stream)
            dsum = lora_sum_bf16([r[0] for r in res], stream=stream)
            return dsum, [(r[1], r[2]) for r in res]
        dsum, res = _tp.tp_linear_bwd_column_group(self.comm, [self.specs[p] for p in names], probs,
                                                   [self.alpha] * len(names), stream=stream)
        return dsum, [(r[1], r[2]) for r in res]

    # ----------------------------------------------------------------- backward
    def backward(self, dout, stream=None):
        C, P, c = self.ctx, self.P, self.cfg
        T = dout.shape[0]
        grads = {}
        d_a, grads["da_down"], grads["db_down"] = self._row_bwd("down", C["a"], dout, C["hdn"], stream)
        d_g, d_u = lora_swiglu_bwd(C["g"], C["u"], d_a, stream=stream)
        dh2, gu = self._col_group_bwd(("gate", "up"), C["h2"], (d_g, d_u), (C["hg"], C["hu"]), stream)
        (grads["da_gate"], grads["db_gate"]), (grads["da_up"], grads["db_up"]) = gu
        dx2 = lora_rmsnorm_bwd(dh2, C["x2"], P["g2"], C["rstd2"], dres=dout, stream=stream)
        d_attn, grads["da_o"], grads["db_o"] = self._row_bwd("o", C["attn"], dx2, C["ho"], stream)
        d4 = d_attn.view(T, self.heads, self.D).transpose(0, 1).unsqueeze(0)
        dq4, dk4, dv4 = torch.autograd.grad(C["att4"], (C["qd"], C["kd"], C["vd"]), d4)
        dq, dk, dv = (t[0].transpose(0, 1).reshape(T, self.heads * self.D).contiguous() for t in (dq4, dk4, dv4))
        lora_rope(dq, self.heads, self.D, c["theta"], inverse=True, stream=stream)
        lora_rope(dk, self.heads, self.D, c["theta"], inverse=True, stream=stream)
        dh1, qkv = self._col_group_bwd(("q", "k", "v"), C["h1"], (dq, dk, dv), (C["hq"], C["hk"], C["hv"]), stream)
        for p, (da, db) in zip(("q", "k", "v"), qkv):
            grads["da_" + p], grads["db_" + p] = da, db
        dx = lora_rmsnorm_bwd(dh1, C["x"], P["g1"], C["rstd1"], dres=dx2, stream=stream)
        self.ctx = None
        return dx, grads


def layer_flops(T, d, f, heads, head_dim, r):
    """Algorithmic FLOPs of one layer fwd + bwd: the seven LoRA linears (4 T m n +
    6 T r (m + n) each, no dW0) plus causal attention (QK^T and PV: 2 x 2 T^2 d / 2
    forward, twice that backward)."""
    shapes = [(d, d)] * 4 + [(f, d), (f, d), (d, f)]
    lin = sum(4 * T * m * n + 6 * T * r * (m + n) for m, n in shapes)
    att_fwd = 2 * 2 * T * T * heads * head_dim / 2
    return lin + 3 * att_fwd

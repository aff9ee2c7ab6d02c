"""fp64 CPU oracle of one Llama-2 decoder layer with LoRA on all seven
projections.  TEST INFRASTRUCTURE ONLY: only tests/ and
bench.py's reference legs may import it; the product package never does.

Plain PyTorch CPU ops in float64, written in the order of the definitions:
  Llama-2 block (JORA builds on a Llama-2 implementation; the
  block structure is the Llama-2 architecture's -- the paper does not restate
  it, R18):
    h1  = RMSNorm(x; g1)                      y = g * x / sqrt(mean(x^2) + eps)
    q, k, v = LoRA(h1; W_q/k/v, A, B)         y = x W0^T + s (x A^T) B^T  (Eq. 1)
    q, k = RoPE(q), RoPE(k)                   pairs (i, i + D/2), angle t theta^(-2i/D)
    o   = softmax(q k^T / sqrt(D) + causal mask) v     per head
    x2  = x + LoRA(o; W_o ...)
    a   = silu(LoRA(h2; W_gate)) * LoRA(h2; W_up),  h2 = RMSNorm(x2; g2)
    out = x2 + LoRA(a; W_down)
The backward is torch.autograd of this forward (the definition of the
gradient); W0 and the norm weights are frozen, so the
gradients are dx and (dA, dB) of the seven adapters.  Pins (tests/
test_oracle_layer_pins.py) check each piece against closed forms and the
whole gradient against central finite differences.
"""
from __future__ import annotations

import math

import torch

PROJ = ("q", "k", "v", "o", "gate", "up", "down")


def rmsnorm(x, g, eps):
    return g * (x * torch.rsqrt((x * x).mean(dim=-1, keepdim=True) + eps))


def rope(q, heads, D, theta, pos0=0):
    T = q.shape[0]
    half = D // 2
    i = torch.arange(half, dtype=torch.float64)
    inv = theta ** (-2.0 * i / D)
    ang = (pos0 + torch.arange(T, dtype=torch.float64))[:, None] * inv[None, :]
    cos, sin = ang.cos()[:, None, :], ang.sin()[:, None, :]
    qh = q.reshape(T, heads, D)
    a, b = qh[..., :half], qh[..., half:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1).reshape(T, heads * D)


def causal_attention(q, k, v, heads, D):
    T = q.shape[0]
    qh, kh, vh = (t.reshape(T, heads, D).transpose(0, 1) for t in (q, k, v))   # [H, T, D]
    scores = qh @ kh.transpose(1, 2) / math.sqrt(D)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool), diagonal=1)
    scores = scores.masked_fill(mask, float("-inf"))
    p = torch.softmax(scores, dim=-1)
    return (p @ vh).transpose(0, 1).reshape(T, heads * D)


def swiglu(gate, up):
    return gate * torch.sigmoid(gate) * up


def lora(x, w0, a, b, alpha):
    s = alpha / a.shape[0]
    return x @ w0.T + s * ((x @ a.T) @ b.T)


def layer_forward(x, P, cfg):
    """x [T, d]; P: dict of fp64 tensors (w0_*, a_*, b_*, g1, g2); cfg: heads, head_dim,
    eps, theta, alpha."""
    H, D, eps, th, al = cfg["heads"], cfg["head_dim"], cfg["eps"], cfg["theta"], cfg["alpha"]
    L = lambda name, inp: lora(inp, P["w0_" + name], P["a_" + name], P["b_" + name], al)  # noqa: E731
    h1 = rmsnorm(x, P["g1"], eps)
    q, k, v = L("q", h1), L("k", h1), L("v", h1)
    q, k = rope(q, H, D, th), rope(k, H, D, th)
    o = causal_attention(q, k, v, H, D)
    x2 = x + L("o", o)
    h2 = rmsnorm(x2, P["g2"], eps)
    a = swiglu(L("gate", h2), L("up", h2))
    return x2 + L("down", a)


def layer_forward_backward(x, dout, P, cfg):
    """Returns (out, dx, {"da_<p>", "db_<p>"}) for the seven projections (fp64)."""
    x = x.clone().requires_grad_(True)
    Q = {k: (v.clone().requires_grad_(True) if k[:2] in ("a_", "b_") else v) for k, v in P.items()}
    out = layer_forward(x, Q, cfg)
    names = [f"{ab}_{p}" for p in PROJ for ab in ("a", "b")]
    grads = torch.autograd.grad(out, [x] + [Q[nm] for nm in names], dout)
    return out.detach(), grads[0], {"d" + nm: g for nm, g in zip(names, grads[1:])}

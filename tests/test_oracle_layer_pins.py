"""Pins of the decoder-layer oracle (oracle/layer.py) against
closed forms, brute-force loops and finite differences -- none re-types the
oracle's formula."""
import math

import numpy as np
import pytest
import torch

from oracle import layer as OL
from synth import bf16_bits_to_f64, make_layer_inputs

F64 = torch.float64


def test_rmsnorm_closed_forms():
    g = torch.tensor([1.0, 2.0, -3.0, 0.5], dtype=F64)
    # a constant row c * 1 has rms |c|: the output is g * sign(c) (eps = 0)
    for c in (0.3, -7.0):
        assert torch.allclose(OL.rmsnorm(torch.full((1, 4), c, dtype=F64), g, 0.0), g * math.copysign(1.0, c), rtol=0, atol=1e-15)
    x = torch.tensor([[3.0, 4.0, 0.0, 0.0]], dtype=F64)     # mean square 25/4 -> rms 2.5
    assert torch.allclose(OL.rmsnorm(x, torch.ones(4, dtype=F64), 0.0), x / 2.5, rtol=0, atol=1e-15)
    # eps: mean square 0 -> x / sqrt(eps)
    assert torch.allclose(OL.rmsnorm(torch.tensor([[1e-3, 0, 0, 0]], dtype=F64), torch.ones(4, dtype=F64), 0.25),
                          torch.tensor([[2e-3, 0, 0, 0]], dtype=F64), rtol=1e-12)


def test_rope_closed_forms():
    # one pair (D = 2): angle = t exactly (theta^0 = 1); (1, 0) -> (cos t, sin t)
    T = 5
    q = torch.tensor([[1.0, 0.0]] * T, dtype=F64)
    r = OL.rope(q, 1, 2, 10000.0)
    for t in range(T):
        assert abs(r[t, 0] - math.cos(t)) < 1e-15 and abs(r[t, 1] - math.sin(t)) < 1e-15
    # position 0 is the identity; the pair norms are preserved
    g = torch.Generator().manual_seed(0)
    q = torch.randn(7, 3 * 16, generator=g, dtype=F64)
    r = OL.rope(q, 3, 16, 500.0)
    assert torch.equal(r[0], q[0])
    qh, rh = q.reshape(7, 3, 2, 8), r.reshape(7, 3, 2, 8)
    assert torch.allclose((qh ** 2).sum(2), (rh ** 2).sum(2), rtol=1e-13)
    # relative positions: <RoPE(q)_t1, RoPE(k)_t2> depends on t1 - t2 only (same q, k rows at all t)
    qq = torch.randn(1, 16, generator=g, dtype=F64).repeat(6, 1)
    kk = torch.randn(1, 16, generator=g, dtype=F64).repeat(6, 1)
    rq, rk = OL.rope(qq, 1, 16, 10000.0), OL.rope(kk, 1, 16, 10000.0)
    assert abs(float(rq[4] @ rk[1] - rq[3] @ rk[0])) < 1e-12
    assert abs(float(rq[5] @ rk[5] - rq[0] @ rk[0])) < 1e-12


def test_attention_brute_force():
    g = torch.Generator().manual_seed(1)
    T, H, D = 5, 2, 4
    q, k, v = (torch.randn(T, H * D, generator=g, dtype=F64) for _ in range(3))
    o = OL.causal_attention(q, k, v, H, D)
    for h in range(H):
        sl = slice(h * D, (h + 1) * D)
        for t in range(T):
            s = [sum(float(q[t, sl][i] * k[u, sl][i]) for i in range(D)) / math.sqrt(D) for u in range(t + 1)]
            mx = max(s)
            w = [math.exp(x - mx) for x in s]
            ref = [sum(w[u] * float(v[u, sl][i]) for u in range(t + 1)) / sum(w) for i in range(D)]
            assert np.allclose(o[t, sl].numpy(), ref, rtol=1e-12, atol=1e-14)
    # T = 1: the output is v; equal keys: the causal prefix mean of v
    assert torch.allclose(OL.causal_attention(q[:1], k[:1], v[:1], H, D), v[:1], rtol=0, atol=1e-15)
    kc = torch.ones(T, H * D, dtype=F64)
    qz = torch.zeros(T, H * D, dtype=F64)
    pm = torch.cumsum(v, 0) / torch.arange(1, T + 1, dtype=F64)[:, None]
    assert torch.allclose(OL.causal_attention(qz, kc, v, H, D), pm, rtol=1e-13)


def test_swiglu_closed_form():
    g = torch.tensor([0.0, 1.0, -2.0, 30.0], dtype=F64)
    u = torch.tensor([5.0, 2.0, 3.0, 0.5], dtype=F64)
    ref = [0.0, 2.0 / (1 + math.exp(-1.0)), 3.0 * -2.0 / (1 + math.exp(2.0)), 0.5 * 30.0 / (1 + math.exp(-30.0))]
    assert np.allclose(OL.swiglu(g, u).numpy(), ref, rtol=1e-15)


def _layer_small(seed=3):
    T, d, f, H, r = 6, 32, 48, 2, 4
    bits = make_layer_inputs(T, d, f, H, r, seed=seed)
    P = {k: torch.from_numpy(bf16_bits_to_f64(v)) for k, v in bits.items()}
    cfg = dict(heads=H, head_dim=d // H, eps=1e-5, theta=10000.0, alpha=8.0)
    return P, cfg


def test_zero_weights_is_identity():
    P, cfg = _layer_small()
    Z = {k: (torch.zeros_like(v) if k.startswith(("w0_", "a_", "b_")) else v) for k, v in P.items()}
    out, dx, grads = OL.layer_forward_backward(P["x"], P["dout"], Z, cfg)
    assert torch.equal(out, P["x"]) and torch.equal(dx, P["dout"])
    assert all(float(g.abs().max()) == 0.0 for g in grads.values())   # B = A = 0: no LoRA gradient


def test_gradients_match_finite_differences():
    P, cfg = _layer_small()
    x, dout = P["x"], P["dout"]
    out, dx, grads = OL.layer_forward_backward(x, dout, P, cfg)
    loss = lambda Q, xx: float((OL.layer_forward(xx, Q, cfg) * dout).sum())  # noqa: E731
    eps = 1e-6
    rng = np.random.default_rng(0)
    for _ in range(6):   # dx entries
        t, c = int(rng.integers(x.shape[0])), int(rng.integers(x.shape[1]))
        xp, xm = x.clone(), x.clone()
        xp[t, c] += eps
        xm[t, c] -= eps
        fd = (loss(P, xp) - loss(P, xm)) / (2 * eps)
        assert abs(fd - float(dx[t, c])) <= 1e-6 * (1 + abs(fd))
    for name in ("a_q", "b_v", "a_o", "b_gate", "a_down", "b_k"):   # adapter entries of several projections
        for _ in range(2):
            idx = tuple(int(rng.integers(s)) for s in P[name].shape)
            Qp = dict(P); Qm = dict(P)
            Qp[name] = P[name].clone(); Qm[name] = P[name].clone()
            Qp[name][idx] += eps
            Qm[name][idx] -= eps
            fd = (loss(Qp, x) - loss(Qm, x)) / (2 * eps)
            assert abs(fd - float(grads["d" + name][idx])) <= 1e-6 * (1 + abs(fd)), name

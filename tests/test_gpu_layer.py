"""Llama-2 decoder layer with LoRA on all seven projections (
paper_2403_11366_b200/layer.py) against the fp64 oracle (oracle/layer.py) on the
same bf16 inputs: the layer output, dx and dA / dB of every adapter.  Plus the
pieces alone: RMSNorm fwd / bwd, RoPE (and its inverse), SwiGLU fwd / bwd, the
bf16 sum.

Tolerances: the layer chains ~12 bf16 roundings (norm outputs,
projections, RoPE, attention -- whose probabilities cuDNN keeps in bf16 --, the
SwiGLU product, residual sums), against 2 for one LoRA linear: relF <= 2e-2 for
the output and dx, <= 4e-2 for the adapter gradients (twice the linear's)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import layer as OL  # noqa: E402
from synth import bf16_bits_to_f64, make_layer_inputs  # noqa: E402
from tests.gpu_util import dev_bf16, host_f64, relF  # noqa: E402

TOL_LAYER_OUT, TOL_LAYER_GRAD = 2e-2, 4e-2


def _f64(bits):
    return torch.from_numpy(bf16_bits_to_f64(bits))


@pytest.mark.parametrize("T,d,f,H,r", [(256, 512, 1376, 4, 8), (300, 256, 704, 2, 16)])
def test_layer_fwd_bwd_matches_oracle(T, d, f, H, r):
    from paper_2403_11366_b200.layer import LlamaLayerLoRA
    bits = make_layer_inputs(T, d, f, H, r, seed=77 + T)
    cfg = dict(heads=H, head_dim=d // H, eps=1e-5, theta=10000.0, alpha=16.0, ffn=f)
    P64 = {k: _f64(v) for k, v in bits.items()}
    out_o, dx_o, g_o = OL.layer_forward_backward(P64["x"], P64["dout"], P64, cfg)
    params = {k: dev_bf16(v) for k, v in bits.items() if k not in ("x", "dout")}
    layer = LlamaLayerLoRA(params, cfg)
    out = layer.forward(dev_bf16(bits["x"]))
    dx, grads = layer.backward(dev_bf16(bits["dout"]))
    torch.cuda.synchronize()
    errs = {"out": relF(host_f64(out), out_o.numpy()), "dx": relF(host_f64(dx), dx_o.numpy())}
    for k, v in g_o.items():
        errs[k] = relF(host_f64(grads[k]), v.numpy())
    print(errs)
    assert errs["out"] <= TOL_LAYER_OUT and errs["dx"] <= TOL_LAYER_OUT
    for k in g_o:
        assert errs[k] <= TOL_LAYER_GRAD, (k, errs[k])


def test_layer_pieces_match_oracle():
    import paper_2403_11366_b200 as L
    g = np.random.default_rng(3)
    T, d, H, D = 130, 384, 3, 128
    from synth import f32_to_bf16_bits
    xb, rb, gb, dyb = (f32_to_bf16_bits(g.standard_normal(s).astype(np.float32)) for s in ((T, d), (T, d), (d,),
                                                                                       (T, d)))
    x, res, gw, dy = (dev_bf16(b) for b in (xb, rb, gb, dyb))
    x64, r64, g64, dy64 = (torch.from_numpy(bf16_bits_to_f64(b)) for b in (xb, rb, gb, dyb))
    # RMSNorm with the residual add (the residual stream is bf16: x2 rounded once)
    x2 = torch.empty_like(x)
    y, rstd = L.lora_rmsnorm_fwd(x, gw, 1e-5, res=res, x2_out=x2)
    x2_64 = host_f64(x2)
    assert np.array_equal(x2_64, host_f64((x.float() + res.float()).bfloat16()))
    y_o = OL.rmsnorm(torch.from_numpy(x2_64), g64, 1e-5).numpy()
    assert relF(host_f64(y), y_o) <= 1e-2
    # RMSNorm backward vs autograd of the oracle's definition (g frozen)
    xx = torch.from_numpy(x2_64).requires_grad_(True)
    (gx,) = torch.autograd.grad(OL.rmsnorm(xx, g64, 1e-5), xx, dy64)
    dx = L.lora_rmsnorm_bwd(dy, x2, gw, rstd, dres=res)
    assert relF(host_f64(dx), (gx + r64).numpy()) <= 1e-2
    # RoPE forward and inverse (the backward is the transpose of the rotation)
    q = x.clone()
    L.lora_rope(q, H, D, 10000.0)
    assert relF(host_f64(q), OL.rope(x64, H, D, 10000.0).numpy()) <= 1e-2
    L.lora_rope(q, H, D, 10000.0, inverse=True)
    assert relF(host_f64(q), x64.numpy()) <= 1e-2
    # SwiGLU forward / backward vs autograd of the definition
    gt = torch.from_numpy(host_f64(x)).requires_grad_(True)
    ut = torch.from_numpy(host_f64(res)).requires_grad_(True)
    a_o = OL.swiglu(gt, ut)
    dg_o, du_o = torch.autograd.grad(a_o, (gt, ut), dy64)
    a = L.lora_swiglu_fwd(x, res)
    dg, du = L.lora_swiglu_bwd(x, res, dy)
    assert relF(host_f64(a), a_o.detach().numpy()) <= 1e-2
    assert relF(host_f64(dg), dg_o.numpy()) <= 1e-2 and relF(host_f64(du), du_o.numpy()) <= 1e-2
    # the bf16 sum: one rounding of the fp32 sum
    s = L.lora_sum_bf16([x, res, dy])
    ref = (x.float() + res.float() + dy.float()).bfloat16()
    torch.cuda.synchronize()
    assert torch.equal(s, ref)


def test_layer_tp_path_one_rank():
    """The TP composition (column groups through lora_tp_linear_bwd_column_group,
    row projections through lora_tp_linear_fwd / bwd, real 1-rank NCCL
    collectives) gives the same layer as the single-GPU composition bitwise."""
    from paper_2403_11366_b200 import tp
    from paper_2403_11366_b200.layer import LlamaLayerLoRA
    T, d, f, H, r = 256, 256, 704, 2, 8
    bits = make_layer_inputs(T, d, f, H, r, seed=5)
    cfg = dict(heads=H, head_dim=d // H, eps=1e-5, theta=10000.0, alpha=16.0, ffn=f)
    params = {k: dev_bf16(v) for k, v in bits.items() if k not in ("x", "dout")}
    x, dout = dev_bf16(bits["x"]), dev_bf16(bits["dout"])
    ref = LlamaLayerLoRA(params, cfg)
    out1 = ref.forward(x)
    dx1, g1 = ref.backward(dout)
    comm = tp.LoraComm()
    try:
        lay = LlamaLayerLoRA(params, cfg, comm=comm)
        out2 = lay.forward(x)
        dx2, g2 = lay.backward(dout)
        torch.cuda.synchronize()
    finally:
        comm.close()
    assert torch.equal(out1, out2) and torch.equal(dx1, dx2)
    for k in g1:
        assert torch.equal(g1[k], g2[k]), k


def _layer_cases(n_cases=6, seed=555):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        H = int(rng.choice([1, 2, 4]))
        hd = int(rng.choice([64, 128]))
        out.append((int(rng.integers(16, 420)), H * hd, 8 * int(rng.integers(8, 200)), H, int(rng.integers(1, 33))))
    return out


@pytest.mark.parametrize("T,d,f,H,r", _layer_cases())
def test_layer_fuzz(T, d, f, H, r):
    """Seeded random layer configurations (T, heads, head_dim 64 / 128, ffn, rank) through
    the same checks as test_layer_fwd_bwd_matches_oracle."""
    test_layer_fwd_bwd_matches_oracle(T, d, f, H, r)

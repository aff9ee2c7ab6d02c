"""GPU parity of the fused adapter update (lora_adam_step)
against the fp64 oracle (oracle.adam_step, pinned in test_oracle_adam_pins)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2403_11366_b200 as L
    L.lora_device_check()
    return L


def _rand_tensors(shapes, seed, master=True):
    g = torch.Generator().manual_seed(seed)
    out = []
    for sh in shapes:
        w = (torch.randn(sh, generator=g) * 0.02).float()
        out.append(dict(master=w.cuda() if master else None, param=w.to(torch.bfloat16).cuda(),
                        m=torch.zeros(sh).cuda(), v=torch.zeros(sh).cuda(),
                        w64=w.double().numpy() if master else w.to(torch.bfloat16).double().numpy(),
                        m64=np.zeros(sh), v64=np.zeros(sh)))
    return out


@pytest.mark.parametrize("use_master", [True, False])
def test_adam_trajectory_matches_oracle(oracle_mod, L, use_master):
    """Five steps on the adapters of a q/v pair (A [r,n], B [m,r]) plus odd
    shapes, one launch per step; fp32 state vs the fp64 oracle."""
    shapes = [(8, 4096), (4096, 8), (16, 136), (200, 4)]
    ts = _rand_tensors(shapes, 11, master=use_master)
    gen = torch.Generator().manual_seed(12)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    for step in range(1, 6):
        grads = [torch.randn(sh, generator=gen) * (0.1 * step) for sh in shapes]
        L.lora_adam_step([(t["param"], g.cuda(), t["m"], t["v"], t["master"]) for t, g in zip(ts, grads)], step, lr,
                         (b1, b2), eps)
        assert L.lora_last_launch_count() == 1
        torch.cuda.synchronize()
        for t, g in zip(ts, grads):
            # the hyper-parameters cross the C ABI as fp32: give the oracle those exact values
            f32 = lambda z: float(np.float32(z))  # noqa: E731
            t["w64"], t["m64"], t["v64"] = oracle_mod.adam_step(t["w64"], g.double().numpy(), t["m64"], t["v64"],
                                                                step, f32(lr), f32(b1), f32(b2), f32(eps))
            if not use_master:   # the state is the bf16 param itself: follow the GPU's rounding
                t["w64"] = torch.from_numpy(t["w64"]).float().to(torch.bfloat16).double().numpy()
    # fp32 state vs fp64: |g| <= ~2.5 here, so the moments carry ~1e-7 absolute
    # rounding (cancellation makes small m relatively noisier) and theta, whose
    # step is ~lr per iteration, ~1e-3 lr; a formula error moves theta by ~lr.
    for t in ts:
        np.testing.assert_allclose(t["m"].cpu().double().numpy(), t["m64"], rtol=1e-5, atol=2e-7)
        np.testing.assert_allclose(t["v"].cpu().double().numpy(), t["v64"], rtol=1e-5, atol=1e-8)
        p = t["param"].cpu().double().numpy()
        if use_master:
            w = t["master"].cpu()
            np.testing.assert_allclose(w.double().numpy(), t["w64"], rtol=0, atol=5e-3 * lr)
            assert torch.equal(t["param"].cpu(), w.to(torch.bfloat16))     # param = RNE(master)
        else:
            frac = np.mean(p == t["w64"])
            assert frac >= 0.99, frac
            np.testing.assert_allclose(p, t["w64"], rtol=2 ** -7, atol=1e-6)


def test_adam_zero_grad_and_validation(L):
    ts = _rand_tensors([(8, 64)], 3)
    t = ts[0]
    before = t["param"].clone()
    L.lora_adam_step([(t["param"], torch.zeros(8, 64).cuda(), t["m"], t["v"], t["master"])], 1, 0.1)
    torch.cuda.synchronize()
    assert torch.equal(t["param"], before)
    with pytest.raises(L.LoraError):
        L.lora_adam_step([(t["param"], torch.zeros(8, 64).cuda(), t["m"], t["v"], t["master"])], 0, 0.1)
    odd = torch.zeros(6, dtype=torch.bfloat16).cuda()
    with pytest.raises(L.LoraError):
        L.lora_adam_step([(odd, torch.zeros(6).cuda(), torch.zeros(6).cuda(), torch.zeros(6).cuda(), None)], 1, 0.1)


def test_lora_training_loop_reduces_loss(L):
    """End to end through the C ABI (fwd -> bwd -> Adam on A, B; W0 frozen):
    fit a rank-r update of a frozen 512x512 projection; the LoRA path alone
    must drive the loss down by > 10x while W0 stays bit-identical."""
    torch.manual_seed(0)
    T, n, m, r, alpha = 512, 512, 512, 8, 16.0
    x = torch.randn(T, n).cuda().to(torch.bfloat16)
    w0 = (torch.randn(m, n) / n ** 0.5).cuda().to(torch.bfloat16)
    w0_before = w0.clone()
    delta = (torch.randn(m, r) @ torch.randn(r, n) / (n ** 0.5 * r)).cuda()
    y_t = (x.float() @ (w0.float() + delta).t())
    a_master = (torch.randn(r, n) * 0.02).cuda()          # B = 0 at start
    b_master = torch.zeros(m, r).cuda()
    a, b = a_master.to(torch.bfloat16), b_master.to(torch.bfloat16)
    st = {k: (torch.zeros_like(t), torch.zeros_like(t)) for k, t in (("a", a_master), ("b", b_master))}
    losses = []
    for step in range(1, 61):
        y, h = L.lora_linear_fwd(x, w0, a, b, alpha)
        diff = y.float() - y_t
        losses.append(float((diff * diff).mean()))
        dy = (2.0 * diff / diff.numel()).to(torch.bfloat16)
        _, da, db = L.lora_linear_bwd(x, w0, a, b, dy, alpha, h_saved=h, want_dx=False)
        L.lora_adam_step([(a, da, *st["a"], a_master), (b, db, *st["b"], b_master)], step, 2e-3)
    torch.cuda.synchronize()
    assert losses[-1] < 0.1 * losses[0], (losses[0], losses[-1])
    assert torch.equal(w0, w0_before)


@pytest.mark.parametrize("seed", range(4))
def test_adam_fuzz(oracle_mod, L, seed):
    """Seeded random adapter sets (1-12 tensors of r x n / m x r shapes, element
    counts multiples of 8), hyper-parameters and gradient scales: three steps of
    one launch each vs the fp64 oracle (fp32 master state)."""
    rng = np.random.default_rng(900 + seed)
    shapes = []
    for _ in range(int(rng.integers(1, 13))):
        r, d = int(rng.integers(1, 65)), 8 * int(rng.integers(1, 600))
        shapes.append((r, d) if rng.integers(0, 2) else (d, r))
    ts = _rand_tensors(shapes, 50 + seed)
    lr, b1, b2 = float(rng.choice([1e-4, 1e-3, 3e-3])), float(rng.choice([0.8, 0.9])), float(rng.choice([0.99, 0.999]))
    eps = 1e-8
    gen = torch.Generator().manual_seed(60 + seed)
    f32 = lambda z: float(np.float32(z))  # noqa: E731
    for step in range(1, 4):
        grads = [torch.randn(sh, generator=gen) * float(rng.choice([1e-3, 0.1, 1.0])) for sh in shapes]
        L.lora_adam_step([(t["param"], g.cuda(), t["m"], t["v"], t["master"]) for t, g in zip(ts, grads)], step, lr,
                         (b1, b2), eps)
        torch.cuda.synchronize()
        for t, g in zip(ts, grads):
            t["w64"], t["m64"], t["v64"] = oracle_mod.adam_step(t["w64"], g.double().numpy(), t["m64"], t["v64"],
                                                                step, f32(lr), f32(b1), f32(b2), f32(eps))
    for t in ts:
        scale = max(float(np.abs(t["m64"]).max()), 1e-12)
        np.testing.assert_allclose(t["m"].cpu().double().numpy(), t["m64"], rtol=1e-5, atol=1e-6 * scale)
        np.testing.assert_allclose(t["master"].cpu().double().numpy(), t["w64"], rtol=0, atol=5e-3 * lr)
        assert torch.equal(t["param"].cpu(), t["master"].cpu().to(torch.bfloat16))

"""GPU parity: the sm_100a path (through the C ABI) against the fp64 oracle on
the same seeded bf16 inputs.  Tolerances from north_star (BASELINE.json):
relative Frobenius error <= 1e-2 for y, dX and <= 2e-2 for dA, dB; bit-exact
where the arithmetic is exact (integer-valued inputs)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import bf16_bits_to_f64, f32_to_bf16_bits, make_lora_inputs  # noqa: E402
from tests.gpu_util import (TOL_GRAD, TOL_OUT, bits_of, dev_bf16, host_f64, relF,  # noqa: E402
                            rne_bf16_f64)


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2403_11366_b200 as L
    L.lora_device_check()
    return L


def _run(L, d, alpha, bias=None, h_saved=True, want_dx=True):
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    bb = dev_bf16(bias) if bias is not None else None
    y, h = L.lora_linear_fwd(x, w0, a, b, alpha, bias=bb)
    dx, da, db = L.lora_linear_bwd(x, w0, a, b, dy, alpha, h_saved=h if h_saved else None,
                                   want_dx=want_dx)
    torch.cuda.synchronize()
    return dict(y=y, h=h, dx=dx, da=da, db=db)


def _check_against_oracle(oracle_mod, L, d, alpha, rows=None, bias=None, **kw):
    out = _run(L, d, alpha, bias=bias, **kw)
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, bias=bias, rows=rows)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, rows=rows)
    sel = slice(None) if rows is None else rows
    errs = {
        "y": relF(host_f64(out["y"])[sel], yo),
        "h": relF(host_f64(out["h"])[sel], ho),
        "da": relF(host_f64(out["da"]), go["da"]),
        "db": relF(host_f64(out["db"]), go["db"]),
    }
    if out["dx"] is not None:
        errs["dx"] = relF(host_f64(out["dx"])[sel], go["dx"])
    assert errs["y"] <= TOL_OUT, errs
    assert errs.get("dx", 0.0) <= TOL_OUT, errs
    assert errs["da"] <= TOL_GRAD and errs["db"] <= TOL_GRAD, errs
    assert errs["h"] <= 1e-4, errs  # h is an fp32 accumulation of the same bf16 products
    return out, errs


# ------------------------------------------------------------------ configs
def test_cfg1_parity(oracle_mod, L):
    """BASELINE.json configs[0]: 64 -> 64, r = 4, 128 tokens (alpha = 16, s = 4)."""
    d = make_lora_inputs(128, 64, 64, 4, seed=2403)
    _, errs = _check_against_oracle(oracle_mod, L, d, 16.0)
    print("cfg1 relF", errs)


@pytest.mark.parametrize("shape", [
    (300, 200, 264, 5),     # ragged T, n, m; r < 16
    (1, 8, 8, 1),           # minimum sizes
    (129, 64, 520, 17),     # r_pad = 32, m spans tiles with a ragged tail
    (257, 136, 256, 33),    # r_pad = 64
    (64, 1024, 8, 64),      # max rank, d_out smaller than a tile
    (700, 512, 488, 16),    # several row and column tiles
    (130, 256, 240, 8),     # exactly one BN = 240 column tile
    (256, 72, 1000, 12),    # K smaller than two k-blocks, many column tiles
])
def test_ragged_shapes_and_ranks(oracle_mod, L, shape):
    T, n, m, r = shape
    d = make_lora_inputs(T, n, m, r, seed=100 + r)
    _check_against_oracle(oracle_mod, L, d, 16.0)


def test_cfg2_full_size_sampled_rows(oracle_mod, L):
    """BASELINE.json configs[1] at full size in the bench's launch
    configuration: y, dX checked on sampled rows (first, last, random), dA and
    dB in full."""
    T, n, m, r = 2048, 4096, 4096, 8
    d = make_lora_inputs(T, n, m, r, seed=2403)
    rng = np.random.default_rng(7)
    rows = np.unique(np.concatenate([[0, 1, 127, 128, T - 1], rng.choice(T, 40, replace=False)]))
    _, errs = _check_against_oracle(oracle_mod, L, d, 16.0, rows=rows)
    print("cfg2 relF", errs)


@pytest.mark.parametrize("shape", [(4096, 4096, 11008, 16), (4096, 11008, 4096, 16), (4096, 5120, 13824, 8),
                                   (4096, 8192, 1024, 16)])
def test_layer_set_shapes_sampled_rows(oracle_mod, L, shape):
    """BASELINE.json configs[2..4] projection shapes (7B gate/up and down,
    13B MLP, 70B GQA k/v) at T = 4096: y, dX on sampled rows, dA, dB in full."""
    T, n, m, r = shape
    d = make_lora_inputs(T, n, m, r, seed=300 + r)
    rng = np.random.default_rng(11)
    rows = np.unique(np.concatenate([[0, T - 1], rng.choice(T, 24, replace=False)]))
    _, errs = _check_against_oracle(oracle_mod, L, d, 16.0, rows=rows)
    print(shape, "relF", errs)


# ------------------------------------------------------------------ exact pins
def test_worked_example_embedded_bit_exact(oracle_mod, L):
    """tests/golden/worked_example.json (SPEC.md:324 extended), zero-padded to
    an ABI-legal 128 x 64 -> 64, r = 4: results are small integers, so the GPU
    must match bitwise and every padding element must be exactly 0."""
    from tests.test_oracle_pins import embed_worked_example
    e = embed_worked_example()
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")))["expected"]
    out = _run(L, e, e["alpha"])
    y, dx, da, db = (host_f64(out[k]) for k in ("y", "dx", "da", "db"))
    ey = np.zeros_like(y); ey[0, :2] = g["y"][0]
    edx = np.zeros_like(dx); edx[0, :2] = g["dx"][0]
    eda = np.zeros_like(da); eda[0, :2] = g["da"][0]
    edb = np.zeros_like(db); edb[:2, 0] = [v[0] for v in g["db"]]
    np.testing.assert_array_equal(y, ey)
    np.testing.assert_array_equal(dx, edx)
    np.testing.assert_array_equal(da, eda)
    np.testing.assert_array_equal(db, edb)


def _ternary_certified(oracle_mod, T, n, m, r, alpha):
    s = alpha / r
    for seed in range(50):
        d = make_lora_inputs(T, n, m, r, seed=9000 + seed, dist="ternary")
        _, h = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha)
        go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
        sh, gh = s * h, go["gh"]
        # the bf16 tail operands bf16(s h) and bf16(gh) must be exact
        if np.array_equal(rne_bf16_f64(sh), sh) and np.array_equal(rne_bf16_f64(gh), gh):
            return d
    raise AssertionError("no certified ternary input found")


@pytest.mark.parametrize("shape", [(128, 64, 64, 4), (300, 200, 264, 5), (200, 128, 496, 24)])
def test_integer_exact_bitwise(oracle_mod, L, shape):
    """Ternary inputs {-1, 0, 0, 1} (SURVEY.md 8(c) pin 5): all products and
    sums are integers far below 2^24, so fp32 accumulation is exact and the GPU
    must equal RNE_bf16(oracle) bitwise for y, dX and the oracle exactly for dA,
    dB.  Catches swizzle / layout / indexing bugs a tolerance could hide."""
    T, n, m, r = shape
    alpha = 4.0 * r  # s = 4: a power of two, so s h is an exact integer
    d = _ternary_certified(oracle_mod, T, n, m, r, alpha)
    out = _run(L, d, alpha)
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
    np.testing.assert_array_equal(host_f64(out["y"]), rne_bf16_f64(yo))
    np.testing.assert_array_equal(host_f64(out["h"]), ho)
    np.testing.assert_array_equal(host_f64(out["dx"]), rne_bf16_f64(go["dx"]))
    np.testing.assert_array_equal(host_f64(out["da"]), go["da"])
    np.testing.assert_array_equal(host_f64(out["db"]), go["db"])


def test_b_zero_fresh_adapter(oracle_mod, L):
    """PAPER.md:113 (B initialised to zeros): y and dX equal the base GEMM
    bitwise (the kernel with A = 0 as well), dA == 0 exactly, and y matches
    cuBLAS x W0^T within the output tolerance."""
    T, n, m, r = 384, 512, 640, 8
    d = make_lora_inputs(T, n, m, r, seed=31, zero_b=True)
    out = _run(L, d, 16.0)
    d0 = dict(d, a=np.zeros_like(d["a"]))
    out0 = _run(L, d0, 16.0)
    assert torch.equal(out["y"], out0["y"]) and torch.equal(out["dx"], out0["dx"])
    assert torch.count_nonzero(out["da"]).item() == 0
    x, w0 = dev_bf16(d["x"]), dev_bf16(d["w0"])
    ref = (x.float() @ w0.float().t())
    assert relF(host_f64(out["y"]), host_f64(ref)) <= TOL_OUT
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
    assert relF(host_f64(out["db"]), go["db"]) <= TOL_GRAD


def test_lora_delta_branch(oracle_mod, L):
    """A tolerance on y alone could hide a broken low-rank branch: the GPU's
    y - y|_{B=0} must match the oracle's s h B^T (SURVEY.md 8(c) pin 10)."""
    T, n, m, r = 256, 1024, 768, 8
    d = make_lora_inputs(T, n, m, r, seed=33)
    out = _run(L, d, 16.0)
    out0 = _run(L, dict(d, b=np.zeros_like(d["b"])), 16.0)
    yo, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0)
    yo0, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], np.zeros_like(d["b"]), 16.0)
    assert relF(host_f64(out["y"]) - host_f64(out0["y"]), yo - yo0) <= 2e-2


# ------------------------------------------------------------------ API paths
def test_recompute_h_and_skip_dx(oracle_mod, L):
    """h_saved = NULL recomputes h (K3a); dx = NULL computes gh by K3a."""
    T, n, m, r = 300, 256, 200, 6
    d = make_lora_inputs(T, n, m, r, seed=41)
    _check_against_oracle(oracle_mod, L, d, 16.0, h_saved=False)
    out = _run(L, d, 16.0, want_dx=False)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
    assert out["dx"] is None
    assert relF(host_f64(out["da"]), go["da"]) <= TOL_GRAD
    assert relF(host_f64(out["db"]), go["db"]) <= TOL_GRAD


def test_bias(oracle_mod, L):
    d = make_lora_inputs(200, 128, 136, 4, seed=43, bias=True)
    _check_against_oracle(oracle_mod, L, d, 16.0, bias=d["bias"])


def test_accumulate(L):
    d = make_lora_inputs(256, 128, 192, 8, seed=45)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    _, da1, db1 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h)
    da = da1.clone() * 0.5
    db = db1.clone() * 0.25
    L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_dx=False, da=da, db=db, accumulate=True)
    torch.cuda.synchronize()
    # the second call skips dx, so gh comes from K3a (another fp32 summation order)
    assert torch.allclose(da, 1.5 * da1, rtol=1e-4, atol=1e-4)
    assert torch.allclose(db, 1.25 * db1, rtol=1e-6, atol=1e-6)


def test_zero_tokens(L):
    d = make_lora_inputs(1, 64, 64, 4, seed=47)
    w0, a, b = (dev_bf16(d[k]) for k in ("w0", "a", "b"))
    x = torch.empty((0, 64), dtype=torch.bfloat16, device="cuda")
    dy = torch.empty((0, 64), dtype=torch.bfloat16, device="cuda")
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    da = torch.full((4, 64), 3.0, device="cuda")
    db = torch.full((64, 4), 3.0, device="cuda")
    L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, da=da, db=db)
    torch.cuda.synchronize()
    assert y.shape == (0, 64)
    assert torch.count_nonzero(da).item() == 0 and torch.count_nonzero(db).item() == 0


def test_determinism_and_row_permutation(L):
    """Repeat calls are bitwise identical (fixed reduction orders); token rows
    are independent, so permuting tokens permutes y and dX bitwise."""
    T, n, m, r = 512, 384, 320, 16
    d = make_lora_inputs(T, n, m, r, seed=49)
    o1 = _run(L, d, 16.0)
    o2 = _run(L, d, 16.0)
    for k in ("y", "h", "dx", "da", "db"):
        assert torch.equal(o1[k], o2[k]), k
    perm = np.random.default_rng(3).permutation(T)
    dp = dict(d, x=d["x"][perm], dy=d["dy"][perm])
    op = _run(L, dp, 16.0)
    pt = torch.as_tensor(perm, device="cuda")
    assert torch.equal(op["y"], o1["y"][pt])
    assert torch.equal(op["dx"], o1["dx"][pt])


def test_launch_counts(L):
    d = make_lora_inputs(256, 128, 128, 8, seed=51)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    assert L.lora_last_launch_count() == 1          # fused K1 (r % 8 == 0: TMA reads B directly)
    L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h)
    assert L.lora_last_launch_count() == 2          # fused K2 (computes and splits gh, splits h) + K3
    L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_dx=False)
    assert L.lora_last_launch_count() == 3          # B^T pack + h split, gh row projection (+ split), K3
    d5 = make_lora_inputs(256, 128, 128, 5, seed=51)
    x, w0, a, b = (dev_bf16(d5[k]) for k in ("x", "w0", "a", "b"))
    L.lora_linear_fwd(x, w0, a, b, 16.0)
    assert L.lora_last_launch_count() == 2          # B8 pack (r % 8 != 0) + K1


# ------------------------------------------------------------------ grouped
def test_grouped_equals_single_calls(L):
    """lora_linear_{fwd,bwd}_grouped == the single calls: y, h, dX bitwise (same
    tiles, same k-order, only launched together); dA, dB to fp32 rounding (the
    grouped K3 may split the tokens over a different cluster size, which
    re-associates the fp32 partial sums).  Mixed shapes, T and rank buckets,
    including an r % 8 != 0 problem and one with bias."""
    specs = [(512, 384, 640, 8, False), (300, 256, 136, 8, True), (512, 512, 256, 24, False),
             (128, 64, 72, 5, False)]
    probs, singles = [], []
    for i, (T, n, m, r, bias) in enumerate(specs):
        d = make_lora_inputs(T, n, m, r, seed=70 + i, bias=bias)
        t = {k: dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy")}
        t["bias"] = dev_bf16(d["bias"]) if bias else None
        probs.append(t)
        y, h = L.lora_linear_fwd(t["x"], t["w0"], t["a"], t["b"], 16.0, bias=t["bias"])
        dx, da, db = L.lora_linear_bwd(t["x"], t["w0"], t["a"], t["b"], t["dy"], 16.0, h_saved=h)
        singles.append((y, h, dx, da, db))
    alphas = [16.0] * len(specs)
    fo = L.lora_linear_fwd_grouped([(t["x"], t["w0"], t["a"], t["b"], t["bias"]) for t in probs], alphas)
    bo = L.lora_linear_bwd_grouped([(t["x"], t["w0"], t["a"], t["b"], t["dy"], h) for t, (_, h) in zip(probs, fo)],
                                   alphas)
    torch.cuda.synchronize()
    for (y, h, dx, da, db), (yg, hg), (dxg, dag, dbg) in zip(singles, fo, bo):
        for u, v in ((y, yg), (h, hg), (dx, dxg)):
            assert torch.equal(u, v)
        for u, v in ((da, dag), (db, dbg)):
            torch.testing.assert_close(v, u, rtol=1e-5, atol=1e-5 * float(u.abs().max()))


def test_grouped_shared_input_vs_oracle(oracle_mod, L):
    """q/k/v-style group: several linears read the SAME x, so the grouped K3
    stacks their dA coefficient sets on one pass over x (here r = 64 + 64 + 8
    exceeds one 256-wide MMA, forcing a second job) -- checked against the
    fp64 oracle, with accumulate into existing gradients."""
    T, n = 640, 320
    base = make_lora_inputs(T, n, 8, 8, seed=90)
    x = dev_bf16(base["x"])
    specs = [(192, 64), (136, 64), (256, 8), (72, 5)]
    probs, refs, outs = [], [], []
    for i, (m, r) in enumerate(specs):
        d = make_lora_inputs(T, n, m, r, seed=91 + i)
        d["x"] = base["x"]
        t = {k: dev_bf16(d[k]) for k in ("w0", "a", "b", "dy")}
        ref = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
        da0 = torch.full((r, n), 0.25, device="cuda")
        db0 = torch.full((m, r), -0.5, device="cuda")
        probs.append((x, t["w0"], t["a"], t["b"], t["dy"], None))
        refs.append(ref)
        outs.append((None, da0, db0))
    res = L.lora_linear_bwd_grouped(probs, [16.0] * len(specs), outs=outs, accumulate=True)
    torch.cuda.synchronize()
    for ref, (dx, da, db) in zip(refs, res):
        assert relF(da.cpu().double().numpy() - 0.25, ref["da"]) <= TOL_GRAD
        assert relF(db.cpu().double().numpy() + 0.5, ref["db"]) <= TOL_GRAD
        assert relF(host_f64(dx), ref["dx"]) <= TOL_OUT


def test_grouped_launch_count(L):
    """Two same-bucket problems: one fused launch each for fwd and dX."""
    ts = []
    for i in range(2):
        d = make_lora_inputs(512, 256, 256, 8, seed=80 + i)
        ts.append({k: dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy")})
    fo = L.lora_linear_fwd_grouped([(t["x"], t["w0"], t["a"], t["b"], None) for t in ts], [16.0, 16.0])
    assert L.lora_last_launch_count() == 1
    L.lora_linear_bwd_grouped([(t["x"], t["w0"], t["a"], t["b"], t["dy"], h) for t, (_, h) in zip(ts, fo)],
                              [16.0, 16.0])
    assert L.lora_last_launch_count() == 2      # one grouped dX launch (+ K3 operand split) + one grouped K3


# ------------------------------------------------------------------ merge
# (n, m, r): r % 8 == 0 and r <= 64 run on the tensor cores (lora_merge_mma.cu,
# r_pad 16 / 32 / 64, ragged row and column tiles), the rest on the CUDA cores
@pytest.mark.parametrize("shape", [(64, 64, 4), (4096, 4096, 8), (1000, 520, 33), (520, 1000, 16),
                                   (256, 384, 24), (384, 200, 64), (1024, 8192, 16), (8, 8, 8)])
def test_merge_matches_oracle(oracle_mod, L, shape):
    """lora_merge = RNE_bf16(W0 + s B A) (Eq. 1 line 2): >= 99.9% of elements
    bit-equal to the rounded fp64 oracle, the rest within one bf16 ulp."""
    n, m, r = shape
    d = make_lora_inputs(1, n, m, r, seed=53)
    w0, a, b = (dev_bf16(d[k]) for k in ("w0", "a", "b"))
    wm = L.lora_merge(w0, a, b, 16.0)
    torch.cuda.synchronize()
    ref = rne_bf16_f64(oracle_mod.lora_merge(d["w0"], d["a"], d["b"], 16.0))
    got = host_f64(wm)
    eq = np.mean(got == ref)
    assert eq >= 0.999, eq
    # one bf16 ulp of the result, plus the fp32 evaluation error of W0 + s B A
    # (which matters only where W0 and s B A cancel)
    s = 16.0 / r
    mag = np.abs(bf16_bits_to_f64(d["w0"])) + s * (np.abs(bf16_bits_to_f64(d["b"])) @
                                                   np.abs(bf16_bits_to_f64(d["a"])))
    assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -7 + mag * 2.0 ** -20)
    # in place gives the same bits; W0 unchanged by the out-of-place call
    assert np.array_equal(bits_of(w0), d["w0"])
    w0c = w0.clone()
    L.lora_merge(w0c, a, b, 16.0, w_out=w0c)
    torch.cuda.synchronize()
    assert torch.equal(w0c, wm)


def test_merge_equivalence_forward(L):
    """Eq. 1: the merged weight used as a plain base weight (B = 0) gives the
    adapter forward within tolerance."""
    T, n, m, r = 256, 512, 384, 8
    d = make_lora_inputs(T, n, m, r, seed=55)
    x, w0, a, b = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b"))
    y, _ = L.lora_linear_fwd(x, w0, a, b, 16.0)
    wm = L.lora_merge(w0, a, b, 16.0)
    y2, _ = L.lora_linear_fwd(x, wm, a, torch.zeros_like(b), 16.0)
    torch.cuda.synchronize()
    assert relF(host_f64(y2), host_f64(y)) <= TOL_OUT


def test_frozen_base_untouched(L):
    """fwd + bwd never write W0 (or any input)."""
    d = make_lora_inputs(256, 256, 256, 8, seed=57)
    t = {k: dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy")}
    _run(L, d, 16.0)
    y, h = L.lora_linear_fwd(t["x"], t["w0"], t["a"], t["b"], 16.0)
    L.lora_linear_bwd(t["x"], t["w0"], t["a"], t["b"], t["dy"], 16.0, h_saved=h)
    torch.cuda.synchronize()
    for k, v in t.items():
        assert np.array_equal(bits_of(v), d[k]), k


@pytest.mark.parametrize("split", ["1", "2", "3", "4", "8"])
def test_k3_token_split_paths(oracle_mod, L, split, monkeypatch):
    """Every K3 token split S (cluster size; LORA_K3_S forces it) gives the
    oracle's dA and dB: S = 1 stores straight from TMEM, S > 1 reduces the
    cluster's partials over DSMEM (vectorised for dA and r % 4 == 0 dB, scalar
    for r % 4 != 0), including ranks whose token slice is empty and
    accumulate into existing gradients."""
    monkeypatch.setenv("LORA_K3_S", split)
    for (T, n, m, r) in [(700, 384, 264, 5), (256, 136, 512, 16), (64, 256, 128, 8)]:
        d = make_lora_inputs(T, n, m, r, seed=900 + r)
        x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
        y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
        da0 = torch.full((r, n), 0.5, device="cuda")
        db0 = torch.full((m, r), -1.0, device="cuda")
        _, da, db = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, da=da0, db=db0, accumulate=True)
        torch.cuda.synchronize()
        go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, want_dx=False)
        assert relF(host_f64(da) - 0.5, go["da"]) <= TOL_GRAD, (split, T, n, m, r)
        assert relF(host_f64(db) + 1.0, go["db"]) <= TOL_GRAD, (split, T, n, m, r)


def test_graph_replay_new_inputs(oracle_mod, L):
    """A captured backward (grouped, K2 -> K3 overlapped) replayed with NEW dY and h
    each time: every replay equals the eager call on the same inputs bit for bit
    and the oracle within tolerance.  Guards the per-launch reset of K2's gh flags
    (a flag value frozen into the graph would let later tiles and K3 read the
    previous replay's gh) and K3's wait on them."""
    T, n, m, r, alpha = 1024, 512, 768, 8, 16.0
    base = make_lora_inputs(T, n, m, r, seed=77)
    x, a_q, b_q = dev_bf16(base["x"]), dev_bf16(base["a"]), dev_bf16(base["b"])
    w_q = dev_bf16(base["w0"])
    other = make_lora_inputs(T, n, m, r, seed=78)
    w_v, a_v, b_v = dev_bf16(other["w0"]), dev_bf16(other["a"]), dev_bf16(other["b"])
    dy_q = torch.empty((T, m), dtype=torch.bfloat16, device="cuda")
    dy_v = torch.empty_like(dy_q)
    h_q = torch.empty((T, r), dtype=torch.float32, device="cuda")
    h_v = torch.empty_like(h_q)
    outs = [(torch.empty((T, n), dtype=torch.bfloat16, device="cuda"),
             torch.empty((r, n), dtype=torch.float32, device="cuda"),
             torch.empty((m, r), dtype=torch.float32, device="cuda")) for _ in range(2)]
    probs = [(x, w_q, a_q, b_q, dy_q, h_q), (x, w_v, a_v, b_v, dy_v, h_v)]
    ws = torch.empty(1 << 24, dtype=torch.uint8, device="cuda")

    def load(seed):
        d = make_lora_inputs(T, n, m, r, seed=seed)
        dy_q.copy_(dev_bf16(d["dy"]))
        dy_v.copy_(dev_bf16(make_lora_inputs(T, n, m, r, seed=seed + 500)["dy"]))
        for hh, (ww, aa, bb) in ((h_q, (w_q, a_q, b_q)), (h_v, (w_v, a_v, b_v))):
            _, h = L.lora_linear_fwd(x, ww, aa, bb, alpha)
            hh.copy_(h)
        torch.cuda.synchronize()

    load(1000)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):   # warm-up outside capture (kernel attributes, maps)
        L.lora_linear_bwd_grouped(probs, [alpha, alpha], outs=outs, workspace=ws, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        L.lora_linear_bwd_grouped(probs, [alpha, alpha], outs=outs, workspace=ws, stream=s)
    for seed in (1001, 1002, 1003):
        load(seed)
        g.replay()
        torch.cuda.synchronize()
        got = [[t.clone() for t in o] for o in outs]
        ref = L.lora_linear_bwd_grouped(probs, [alpha, alpha], workspace=ws)
        torch.cuda.synchronize()
        for gi in range(2):
            for t_got, t_ref in zip(got[gi], ref[gi]):
                assert torch.equal(t_got, t_ref), f"replay seed {seed} member {gi}"
        # member q against the oracle
        dq = bits_of(dy_q)
        go = oracle_mod.lora_bwd(base["x"], base["w0"], base["a"], base["b"], dq, alpha)
        assert relF(host_f64(got[0][0]), go["dx"]) <= TOL_OUT
        assert relF(host_f64(got[0][1]), go["da"]) <= TOL_GRAD
        assert relF(host_f64(got[0][2]), go["db"]) <= TOL_GRAD


@pytest.mark.parametrize("shape", [
    (2048, 4096, 4096, 8),   # cfg2: K1 144 tiles, K2 136 tiles on 74 CTA pairs
    (1000, 1032, 2056, 16),  # ragged T, odd column-tile counts, r_pad 16
    (1536, 2048, 3000, 24),  # r_pad 32, a 128-wide last dX tile
])
def test_stream_k_schedule(oracle_mod, L, shape, monkeypatch):
    """With LORA_STREAMK=1, shapes with more tiles than CTA pairs run the stream-K
    tail (split tiles finished by their owner from fp32 partials): y, dX match the oracle on
    sampled rows, dA / dB in full, repeat calls are bitwise equal, and the
    data-parallel schedule (LORA_STREAMK=0) agrees to fp32 re-association."""
    T, n, m, r = shape
    d = make_lora_inputs(T, n, m, r, seed=500 + r)
    rows = np.sort(np.random.default_rng(5).choice(T, 96, replace=False))
    monkeypatch.setenv("LORA_STREAMK", "1")   # opt-in schedule
    out, errs = _check_against_oracle(oracle_mod, L, d, 16.0, rows=rows)
    again = _run(L, d, 16.0)
    for k in ("y", "h", "dx", "da", "db"):
        assert torch.equal(out[k], again[k]), k
    monkeypatch.setenv("LORA_STREAMK", "0")
    dp = _run(L, d, 16.0)
    for k in ("y", "dx"):
        assert relF(host_f64(out[k]), host_f64(dp[k])) <= 2e-3, k   # bf16 outputs: rounding flips only
    for k in ("h", "da", "db"):
        assert relF(host_f64(out[k]), host_f64(dp[k])) <= 1e-5, k


def test_sync_pool_ring_wraps(oracle_mod, L):
    """K2's gh flags come from a recycled ring of a static device pool and are
    zeroed by their last consumer: thousands of eager backward calls (more than
    the ring holds) keep producing the same bits, with and without K3 reading
    the flags, and the result still matches the oracle."""
    T, n, m, r = 384, 256, 512, 8
    d = make_lora_inputs(T, n, m, r, seed=91)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    ref = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h)
    ref_dx_only = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_da=False, want_db=False)
    ws = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    outs = (torch.empty_like(ref[0]), torch.empty_like(ref[1]), torch.empty_like(ref[2]))
    for i in range(9000):   # 16 pool words per call (flags + a done counter): the 131072-word ring wraps
        if i % 2:
            L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dx=outs[0], da=outs[1], db=outs[2], workspace=ws)
        else:
            L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dx=outs[0], want_da=False, want_db=False,
                              workspace=ws)
    torch.cuda.synchronize()
    for u, v in zip(outs, ref):
        assert torch.equal(u, v)
    assert torch.equal(L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_da=False, want_db=False)[0],
                       ref_dx_only[0])
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
    assert relF(host_f64(outs[0]), go["dx"]) <= TOL_OUT


@pytest.mark.parametrize("r", [8, 16, 6])
def test_dx_and_db_without_da_recomputed_h(oracle_mod, L, r):
    """dX and dB requested, dA not, h recomputed (h_saved = NULL): K2 does not
    write a split K3 waits on (the h split comes from the row projection after
    K2), so K3 must not wait on K2's flags (this combination used to
    wait on flags K2 had already reset and trap).  Eager and grouped."""
    T, n, m = 512, 256, 384
    d = make_lora_inputs(T, n, m, r, seed=95 + r)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    dx, da, db = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=None, want_da=False)
    res = L.lora_linear_bwd_grouped([(x, w0, a, b, dy, None)], [16.0], want_da=False)
    torch.cuda.synchronize()
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
    assert da is None
    assert relF(host_f64(dx), go["dx"]) <= TOL_OUT
    assert relF(host_f64(db), go["db"]) <= TOL_GRAD
    assert res[0][1] is None
    assert relF(host_f64(res[0][2]), go["db"]) <= TOL_GRAD
    assert relF(host_f64(res[0][0]), go["dx"]) <= TOL_OUT
    # and dA alone, dB alone, with and without dX, h saved or not
    _, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    for hs in (None, h):
        for want_dx in (True, False):
            for wa, wb in ((True, False), (False, True)):
                o = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=hs, want_dx=want_dx, want_da=wa, want_db=wb)
                torch.cuda.synchronize()
                if wa:
                    assert relF(host_f64(o[1]), go["da"]) <= TOL_GRAD
                if wb:
                    assert relF(host_f64(o[2]), go["db"]) <= TOL_GRAD
                if want_dx:
                    assert relF(host_f64(o[0]), go["dx"]) <= TOL_OUT


def test_grouped_validates_every_problem_before_launch(L):
    """A grouped call whose LAST problem is invalid returns the error with nothing
    enqueued: no launch counted and the first problem's outputs untouched."""
    d = make_lora_inputs(256, 128, 128, 8, seed=97)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y0 = torch.full((256, 128), 7.0, dtype=torch.bfloat16, device="cuda")
    bad_x = torch.empty((256, 128), dtype=torch.bfloat16, device="cuda")[:, 1:].contiguous()   # shape check
    with pytest.raises(ValueError):
        L.lora_linear_fwd_grouped([(x, w0, a, b, None), (bad_x, w0, a, b, None)], [16.0, 16.0])
    # misaligned pointer for problem 1 (passes the binding's checks, fails in the library)
    big = torch.empty(256 * 128 + 8, dtype=torch.bfloat16, device="cuda")
    x_mis = big[1:1 + 256 * 128].view(256, 128)
    with pytest.raises(L.LoraError) as ei:
        L.lora_linear_fwd_grouped([(x, w0, a, b, None), (x_mis, w0, a, b, None)], [16.0, 16.0],
                                  outs=[(y0, None), (None, None)])
    assert "ALIGN" in str(ei.value)
    assert L.lora_last_launch_count() == 0
    torch.cuda.synchronize()
    assert torch.all(y0 == 7.0)
    dx0 = torch.full((256, 128), 7.0, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(L.LoraError):
        L.lora_linear_bwd_grouped([(x, w0, a, b, dy, None), (x_mis, w0, a, b, dy, None)], [16.0, 16.0],
                                  outs=[(dx0, None, None), (None, None, None)])
    assert L.lora_last_launch_count() == 0
    torch.cuda.synchronize()
    assert torch.all(dx0 == 7.0)


def test_captured_sync_words_return_with_the_graph(L):
    """Sync-pool words taken during graph capture belong to the graph and come back
    when it is destroyed: capturing and dropping more graphs than the
    region could hold at once (10000 x 16 words > 131072) keeps working, every
    replay gives the eager result, and the free count returns to its start value."""
    import gc
    T, n, m, r = 256, 128, 256, 8
    d = make_lora_inputs(T, n, m, r, seed=99)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    ref = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h)
    outs = [torch.empty_like(t) for t in ref]
    ws = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dx=outs[0], da=outs[1], db=outs[2], workspace=ws,
                          stream=s)
    torch.cuda.synchronize()
    free0 = L.lora_captured_sync_words_free()
    assert free0 > 0
    for i in range(10000):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dx=outs[0], da=outs[1], db=outs[2], workspace=ws,
                              stream=s)
        assert L.lora_captured_sync_words_free() < free0
        if i % 2500 == 0:
            for t in outs:
                t.zero_()
            g.replay()
            torch.cuda.synchronize()
            for u, v in zip(outs, ref):
                assert torch.equal(u, v)
        del g
        if i % 500 == 499:
            gc.collect()
            torch.cuda.synchronize()
    gc.collect()
    torch.cuda.synchronize()
    import time
    for _ in range(100):   # the runtime runs user-object destructors asynchronously
        if L.lora_captured_sync_words_free() == free0:
            break
        time.sleep(0.05)
    assert L.lora_captured_sync_words_free() == free0

"""GPU parity of the LoRA-dropout path (Listing 3 LORA_DROPOUT, PAPER.md:82;
DESIGN.md reading R7) against the fp64 oracle: the Philox keep mask bit for
bit, then y, h, dX, dA, dB within the north-star tolerances, bitwise where the
arithmetic is exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_lora_inputs  # noqa: E402
from tests.gpu_util import TOL_GRAD, TOL_OUT, dev_bf16, host_f64, relF, rne_bf16_f64  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2403_11366_b200 as L
    L.lora_device_check()
    return L


@pytest.mark.parametrize("T,n,p,seed,offset", [(1, 8, 0.05, 1, 0), (257, 136, 0.05, 2403, 7),
                                               (64, 13, 0.5, 3, 1 << 40), (1000, 4096, 0.3, 2**64 - 1, 2**63 + 5)])
def test_mask_bit_exact(oracle_mod, L, T, n, p, seed, offset):
    got = L.lora_dropout_mask(T, n, (p, seed, offset)).cpu().numpy()
    ref = oracle_mod.dropout_mask(T, n, p, seed, offset)
    np.testing.assert_array_equal(got, ref)


def _run(L, d, alpha, drop, h_saved=True, want_dx=True):
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y, h = L.lora_linear_fwd(x, w0, a, b, alpha, dropout=drop)
    dx, da, db = L.lora_linear_bwd(x, w0, a, b, dy, alpha, h_saved=h if h_saved else None, want_dx=want_dx,
                                   dropout=drop)
    torch.cuda.synchronize()
    return dict(y=y, h=h, dx=dx, da=da, db=db)


@pytest.mark.parametrize("shape", [(300, 200, 264, 5), (129, 64, 520, 17), (257, 136, 256, 33), (64, 1024, 8, 64),
                                   (700, 512, 488, 16), (1, 8, 8, 1), (384, 4096, 1024, 8)])
def test_dropout_parity(oracle_mod, L, shape):
    T, n, m, r = shape
    drop = (0.05, 1000 + r, 3)
    d = make_lora_inputs(T, n, m, r, seed=500 + r)
    out = _run(L, d, 16.0, drop)
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0, dropout=drop)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, dropout=drop)
    errs = {"y": relF(host_f64(out["y"]), yo), "h": relF(host_f64(out["h"]), ho),
            "dx": relF(host_f64(out["dx"]), go["dx"]), "da": relF(host_f64(out["da"]), go["da"]),
            "db": relF(host_f64(out["db"]), go["db"])}
    assert errs["y"] <= TOL_OUT and errs["dx"] <= TOL_OUT, errs
    assert errs["da"] <= TOL_GRAD and errs["db"] <= TOL_GRAD, errs
    assert errs["h"] <= 1e-4, errs
    # the mask really acts: without dropout the adapter terms differ well beyond rounding
    y0, h0 = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0)
    if T * n > 64:
        assert relF(host_f64(out["h"]), h0) > 1e-2


def test_dropout_p0_is_the_plain_call_bitwise(L):
    d = make_lora_inputs(300, 256, 200, 8, seed=601)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y0, h0 = L.lora_linear_fwd(x, w0, a, b, 16.0)
    g0 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h0)
    y1, h1 = L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=(0.0, 9, 9))
    g1 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h1, dropout=(0.0, 9, 9))
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(h0, h1)
    for u, v in zip(g0, g1):
        assert torch.equal(u, v)


def _ternary_certified(oracle_mod, T, n, m, r, alpha, drop):
    s = alpha / r
    for seed in range(60):
        d = make_lora_inputs(T, n, m, r, seed=7000 + seed, dist="ternary")
        _, h = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, dropout=drop)
        go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, dropout=drop)
        if np.array_equal(rne_bf16_f64(s * h), s * h) and np.array_equal(rne_bf16_f64(go["gh"]), go["gh"]):
            return d
    raise AssertionError("no certified ternary input found")


@pytest.mark.parametrize("shape", [(128, 64, 64, 4), (300, 200, 264, 16)])
def test_dropout_integer_exact_bitwise(oracle_mod, L, shape):
    """p = 1/2 (q = 2 exact) on ternary inputs: every intermediate is a small
    integer, so the GPU must match the oracle bitwise (catches a mask applied
    to the wrong element, a missing q, a mask on the frozen path)."""
    T, n, m, r = shape
    alpha, drop = 4.0 * r, (0.5, 42, 5)
    d = _ternary_certified(oracle_mod, T, n, m, r, alpha, drop)
    out = _run(L, d, alpha, drop)
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, dropout=drop)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, dropout=drop)
    np.testing.assert_array_equal(host_f64(out["y"]), rne_bf16_f64(yo))
    np.testing.assert_array_equal(host_f64(out["h"]), ho)
    np.testing.assert_array_equal(host_f64(out["dx"]), rne_bf16_f64(go["dx"]))
    np.testing.assert_array_equal(host_f64(out["da"]), go["da"])
    np.testing.assert_array_equal(host_f64(out["db"]), go["db"])


def test_dropout_recompute_h_and_skip_dx(oracle_mod, L):
    """h_saved = NULL regenerates h from the same mask (bitwise equal grads);
    dX = NULL takes the gh pre-pass path."""
    d = make_lora_inputs(256, 192, 320, 16, seed=603)
    drop = (0.1, 77, 1)
    a1 = _run(L, d, 16.0, drop, h_saved=True)
    a2 = _run(L, d, 16.0, drop, h_saved=False)
    for k in ("dx", "da", "db"):
        assert torch.equal(a1[k], a2[k]), k
    a3 = _run(L, d, 16.0, drop, want_dx=False)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, dropout=drop)
    assert a3["dx"] is None
    assert relF(host_f64(a3["da"]), go["da"]) <= TOL_GRAD
    assert relF(host_f64(a3["db"]), go["db"]) <= TOL_GRAD


def test_dropout_streams_and_determinism(L):
    d = make_lora_inputs(256, 128, 128, 8, seed=604)
    a1 = _run(L, d, 16.0, (0.05, 1, 0))
    a2 = _run(L, d, 16.0, (0.05, 1, 0))
    a3 = _run(L, d, 16.0, (0.05, 1, 1))
    for k in ("y", "h", "dx", "da", "db"):
        assert torch.equal(a1[k], a2[k]), k
    assert not torch.equal(a1["h"], a3["h"])


def test_dropout_cfg2_full_size_sampled_rows(oracle_mod, L):
    """BASELINE.json configs[1] shape with the paper's LORA_DROPOUT = 0.05."""
    T, n, m, r = 2048, 4096, 4096, 8
    drop = (0.05, 2403, 11)
    d = make_lora_inputs(T, n, m, r, seed=2403)
    out = _run(L, d, 16.0, drop)
    rows = np.unique(np.concatenate([[0, 1, 127, 128, T - 1], np.random.default_rng(8).choice(T, 24, replace=False)]))
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0, rows=rows, dropout=drop)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, rows=rows, dropout=drop)
    assert relF(host_f64(out["y"])[rows], yo) <= TOL_OUT
    assert relF(host_f64(out["h"])[rows], ho) <= 1e-4
    assert relF(host_f64(out["dx"])[rows], go["dx"]) <= TOL_OUT
    assert relF(host_f64(out["da"]), go["da"]) <= TOL_GRAD
    assert relF(host_f64(out["db"]), go["db"]) <= TOL_GRAD


def test_dropout_invalid_p(L):
    d = make_lora_inputs(8, 8, 8, 2, seed=605)
    x, w0, a, b = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b"))
    for p in (1.0, -0.1, float("nan")):
        with pytest.raises(L.LoraError):
            L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=(p, 0, 0))


@pytest.mark.parametrize("r,h_saved", [(8, True), (16, False), (5, True)])
def test_grouped_dropout_equals_single_calls(oracle_mod, L, r, h_saved):
    """lora_linear_{fwd,bwd}_grouped_dropout: q/k/v-like members sharing x, each with
    its own mask (seed / offset), one fused launch per kernel -- bitwise the single
    dropout calls, and the oracle's values."""
    T, n = 300, 256
    ms = (256, 128, 136)
    alpha = 16.0
    base = make_lora_inputs(T, n, ms[0], r, seed=620)
    ds, drops = [], []
    for g, m in enumerate(ms):
        d = make_lora_inputs(T, n, m, r, seed=621 + g)
        d["x"] = base["x"]
        ds.append(d)
        drops.append((0.05, 900 + g, 3 * g))
    x = dev_bf16(base["x"])
    ts = [{k: dev_bf16(d[k]) for k in ("w0", "a", "b", "dy")} for d in ds]
    fo = L.lora_linear_fwd_grouped([(x, t["w0"], t["a"], t["b"], None) for t in ts], [alpha] * 3, dropouts=drops)
    go = L.lora_linear_bwd_grouped([(x, t["w0"], t["a"], t["b"], t["dy"], h if h_saved else None)
                                    for t, (_, h) in zip(ts, fo)], [alpha] * 3, dropouts=drops)
    torch.cuda.synchronize()
    for g, (t, d) in enumerate(zip(ts, ds)):
        y1, h1 = L.lora_linear_fwd(x, t["w0"], t["a"], t["b"], alpha, dropout=drops[g])
        dx1, da1, db1 = L.lora_linear_bwd(x, t["w0"], t["a"], t["b"], t["dy"], alpha,
                                          h_saved=h1 if h_saved else None, dropout=drops[g])
        torch.cuda.synchronize()
        assert torch.equal(fo[g][0], y1) and torch.equal(fo[g][1], h1)
        assert torch.equal(go[g][0], dx1) and torch.equal(go[g][1], da1) and torch.equal(go[g][2], db1)
        yo, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, dropout=drops[g])
        gor = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, dropout=drops[g])
        assert relF(host_f64(y1), yo) <= TOL_OUT and relF(host_f64(dx1), gor["dx"]) <= TOL_OUT
        assert relF(host_f64(da1), gor["da"]) <= TOL_GRAD and relF(host_f64(db1), gor["db"]) <= TOL_GRAD


def _pack_bits(mask):
    """uint8 [T, n] keep mask -> the lora_dropout.keep_bits layout: int32 [T, ceil(n/32)],
    bit c of word w of row t = mask[t, 32 w + c] (include/lora.h)."""
    T, n = mask.shape
    nw = (n + 31) // 32
    m = np.zeros((T, nw * 32), dtype=np.uint64)
    m[:, :n] = mask
    words = (m.reshape(T, nw, 32) << np.arange(32, dtype=np.uint64)).sum(axis=2)
    return words.astype(np.uint32).view(np.int32)


@pytest.mark.parametrize("shape", [(300, 200, 264, 5), (257, 136, 256, 16), (33, 40, 64, 33), (384, 4096, 1024, 8)])
def test_keep_bits_forward_writes_backward_reads(oracle_mod, L, shape):
    """lora_dropout.keep_bits / masked_x: the forward writes the oracle's keep mask
    bit for bit (packed 32 per word) and M . x exactly, and a backward that reads
    them instead of redrawing gives bitwise the redrawing backward's dX, dA, dB
    (h saved and recomputed; each buffer alone and both)."""
    T, n, m, r = shape
    d = make_lora_inputs(T, n, m, r, seed=700 + r)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    drop = (0.05, 4242 + r, 11)
    kb = L.dropout_keep_bits(T, n)
    kb.fill_(-1)
    mx = torch.full((T, n), 7.0, dtype=torch.bfloat16, device="cuda")
    y1, h1 = L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=drop + (kb, mx))
    y0, h0 = L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=drop)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(h0, h1)
    mask = oracle_mod.dropout_mask(T, n, *drop)
    np.testing.assert_array_equal(kb.cpu().numpy(), _pack_bits(mask))
    np.testing.assert_array_equal(mx.view(torch.int16).cpu().numpy(),
                                  np.where(mask != 0, d["x"].view(np.int16), np.int16(0)))
    for hs in (h0, None):
        g0 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=hs, dropout=drop)
        for extra in ((kb,), (None, mx), (kb, mx)):
            g1 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=hs, dropout=drop + extra)
            torch.cuda.synchronize()
            for u, v in zip(g0, g1):
                assert torch.equal(u, v)


def test_keep_bits_grouped(oracle_mod, L):
    """Grouped dropout calls with a keep_bits buffer per member: bitwise the calls
    without, and each buffer holds that member's oracle mask."""
    T, n, r = 260, 256, 8
    ms = (256, 136)
    base = make_lora_inputs(T, n, ms[0], r, seed=720)
    x = dev_bf16(base["x"])
    ts, drops, kbs = [], [], []
    for g, m in enumerate(ms):
        dd = make_lora_inputs(T, n, m, r, seed=721 + g)
        ts.append({k: dev_bf16(dd[k]) for k in ("w0", "a", "b", "dy")})
        drops.append((0.05, 77 + g, 5 * g))
        kbs.append((L.dropout_keep_bits(T, n), torch.empty((T, n), dtype=torch.bfloat16, device="cuda")))
    fo0 = L.lora_linear_fwd_grouped([(x, t["w0"], t["a"], t["b"], None) for t in ts], [16.0] * 2, dropouts=drops)
    fo1 = L.lora_linear_fwd_grouped([(x, t["w0"], t["a"], t["b"], None) for t in ts], [16.0] * 2,
                                    dropouts=[dr + kb for dr, kb in zip(drops, kbs)])
    go0 = L.lora_linear_bwd_grouped([(x, t["w0"], t["a"], t["b"], t["dy"], h) for t, (_, h) in zip(ts, fo0)],
                                    [16.0] * 2, dropouts=drops)
    go1 = L.lora_linear_bwd_grouped([(x, t["w0"], t["a"], t["b"], t["dy"], h) for t, (_, h) in zip(ts, fo1)],
                                    [16.0] * 2, dropouts=[dr + kb for dr, kb in zip(drops, kbs)])
    torch.cuda.synchronize()
    for g in range(2):
        assert torch.equal(fo0[g][0], fo1[g][0]) and torch.equal(fo0[g][1], fo1[g][1])
        for u, v in zip(go0[g], go1[g]):
            assert torch.equal(u, v)
        np.testing.assert_array_equal(kbs[g][0].cpu().numpy(), _pack_bits(oracle_mod.dropout_mask(T, n, *drops[g])))


def test_mask_offsets_are_slices_of_the_full_mask(oracle_mod, L):
    """lora_dropout row_offset / col_offset (include/lora.h): the mask of a sub-block
    is the oracle's full mask sliced at that position, bit for bit."""
    T, n, p, seed, off = 300, 200, 0.3, 99, 5
    full = oracle_mod.dropout_mask(T, n, p, seed, off)
    for r0, c0, t, k in ((0, 0, T, n), (17, 8, 100, 64), (129, 136, 171, 64), (299, 192, 1, 8)):
        got = L.lora_dropout_mask(t, k, (p, seed, off, None, None, r0, c0)).cpu().numpy()
        np.testing.assert_array_equal(got, full[r0:r0 + t, c0:c0 + k])


def test_row_sharded_dropout_equals_unsharded_oracle(oracle_mod, L):
    """The tensor-parallel ROW split with dropout, computed shard by shard on one GPU
    (each shard's call with col_offset = its first input column):
    summed y / h partials and concatenated dX / dA equal the UNSHARDED oracle with
    the one mask of the full input; dB from the summed h too."""
    T, n, m, r, alpha = 300, 256, 264, 8, 16.0
    drop = (0.1, 321, 7)
    d = make_lora_inputs(T, n, m, r, seed=731)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    cuts = (0, 96, 256)
    ys, hs = [], []
    for s0, s1 in zip(cuts[:-1], cuts[1:]):
        y, h = L.lora_linear_fwd(x[:, s0:s1].contiguous(), w0[:, s0:s1].contiguous(), a[:, s0:s1].contiguous(), b,
                                 alpha, dropout=drop + (None, None, 0, s0))
        ys.append(host_f64(y))
        hs.append(host_f64(h))
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, dropout=drop)
    h_sum = sum(hs)
    assert relF(h_sum, ho) <= 1e-5
    assert relF(sum(ys), yo) <= TOL_OUT
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, dropout=drop)
    hfull = torch.from_numpy(h_sum.astype(np.float32)).cuda()
    dxs, das = [], []
    for s0, s1 in zip(cuts[:-1], cuts[1:]):
        dx, da, db = L.lora_linear_bwd(x[:, s0:s1].contiguous(), w0[:, s0:s1].contiguous(),
                                       a[:, s0:s1].contiguous(), b, dy, alpha, h_saved=hfull,
                                       dropout=drop + (None, None, 0, s0))
        dxs.append(host_f64(dx))
        das.append(host_f64(da))
        assert relF(host_f64(db), go["db"]) <= TOL_GRAD
    assert relF(np.concatenate(dxs, axis=1), go["dx"]) <= TOL_OUT
    assert relF(np.concatenate(das, axis=1), go["da"]) <= TOL_GRAD


def test_token_slices_with_row_offset_are_bitwise_rows(L):
    """A forward over tokens [t0, t1) with row_offset = t0 gives bitwise the rows
    t0..t1 of the full call (the mask rows follow the offset; K0's per-row sums
    and K1's K-loops do not depend on T)."""
    T, n, m, r = 700, 256, 256, 16
    d = make_lora_inputs(T, n, m, r, seed=741)
    x, w0, a, b = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b"))
    drop = (0.05, 5, 6)
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=drop)
    for t0, t1 in ((0, 256), (256, 512), (512, 700), (123, 457)):
        ys, hs = L.lora_linear_fwd(x[t0:t1].contiguous(), w0, a, b, 16.0, dropout=drop + (None, None, t0, 0))
        torch.cuda.synchronize()
        assert torch.equal(ys, y[t0:t1]) and torch.equal(hs, h[t0:t1]), (t0, t1)

"""Pins for the oracle's LoRA-dropout functions (Listing 3 LORA_DROPOUT = 0.05,
PAPER.md:82; placement and mask definition: DESIGN.md reading R7).

The mask generator is pinned to the published Philox4x32-10 known-answer
vectors and to its counter layout; the dropout forward/backward are pinned by
reduction to the (separately pinned) dropout-free oracle on transformed
inputs -- with p = 1/2 the inverted-dropout factor q = 2 is exact, so the
adapter input xd = q M x is itself a bf16 tensor -- by exact finite
differences (L = <y, G> stays linear in x, A, B for a fixed mask) and by
keep-rate statistics."""
import json
import os

import numpy as np

from synth import bf16_bits_to_f64, f32_to_bf16_bits, make_lora_inputs

KAT = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.json")


def _f(bits):
    return bf16_bits_to_f64(bits)


def test_philox_known_answers(oracle_mod):
    for v in json.load(open(KAT))["vectors"]:
        ctr = [int(c, 16) for c in v["ctr"]]
        key = [int(k, 16) for k in v["key"]]
        assert oracle_mod.philox4x32_10(ctr, key) == tuple(int(o, 16) for o in v["out"])


def test_mask_counter_layout_and_threshold(oracle_mod):
    """M[t,k] = 16-bit draw (k % 8) of Philox((k/8, t, offset_lo, offset_hi), (seed_lo, seed_hi))
    >= floor(p 2^16): word (k % 8) / 2, low half for even k % 8 (R7)."""
    T, n, p, seed, off = 5, 40, 0.3, 0x1234567890ABCDEF, (7 << 32) | 9
    m = oracle_mod.dropout_mask(T, n, p, seed, off)
    thr = oracle_mod.dropout_threshold(p)
    assert thr == int(np.floor(float(np.float32(p)) * 2.0 ** 16))
    assert oracle_mod.dropout_threshold(0.5) == 2 ** 15 and oracle_mod.dropout_threshold(0.0) == 0
    for t in range(T):
        for k in range(n):
            w = oracle_mod.philox4x32_10((k // 8, t, off & 0xFFFFFFFF, off >> 32),
                                         (seed & 0xFFFFFFFF, seed >> 32))
            u = (w[(k % 8) // 2] >> (16 * (k % 2))) & 0xFFFF
            assert m[t, k] == (1 if u >= thr else 0)


def test_mask_statistics_and_streams(oracle_mod):
    T, n = 256, 1024
    for p in (0.05, 0.5):
        m = oracle_mod.dropout_mask(T, n, p, 2403, 0)
        N = T * n
        sigma = np.sqrt(p * (1 - p) / N)
        assert abs((1.0 - m.mean()) - p) < 5 * sigma
    assert oracle_mod.dropout_mask(T, n, 0.0, 1, 2).min() == 1          # p = 0 keeps everything
    a = oracle_mod.dropout_mask(T, n, 0.5, 1, 0)
    b = oracle_mod.dropout_mask(T, n, 0.5, 2, 0)
    c = oracle_mod.dropout_mask(T, n, 0.5, 1, 1)
    for other in (b, c):                                                 # independent streams agree ~half the time
        agree = (a == other).mean()
        assert abs(agree - 0.5) < 5 * np.sqrt(0.25 / (T * n))


def test_p_zero_is_bitwise_the_plain_oracle(oracle_mod):
    T, n, m, r = 19, 40, 24, 5
    d = make_lora_inputs(T, n, m, r, seed=31, bias=True)
    y0, h0 = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0, bias=d["bias"])
    y1, h1 = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0, bias=d["bias"], dropout=(0.0, 5, 6))
    np.testing.assert_array_equal(y0, y1)
    np.testing.assert_array_equal(h0, h1)
    g0 = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
    g1 = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, dropout=(0.0, 5, 6))
    for k in ("dx", "gh", "da", "db"):
        np.testing.assert_array_equal(g0[k], g1[k])


def test_dropout_reduces_to_the_plain_oracle_on_the_masked_input(oracle_mod):
    """p = 1/2 (q = 2 exact): the adapter sees xd = 2 M x (a bf16 tensor), the
    frozen path sees x, and dX's adapter term passes back through q M."""
    T, n, m, r = 33, 48, 40, 6
    alpha, drop = 12.0, (0.5, 77, 3)
    d = make_lora_inputs(T, n, m, r, seed=32)
    M = oracle_mod.dropout_mask(T, n, 0.5, 77, 3)
    xd = f32_to_bf16_bits((2.0 * M * _f(d["x"])).astype(np.float32))
    assert np.array_equal(_f(xd), 2.0 * M * _f(d["x"]))                 # exact
    zeros_b = np.zeros_like(d["b"])
    zeros_w = np.zeros_like(d["w0"])
    zeros_a = np.zeros_like(d["a"])
    y, h = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, dropout=drop)
    _, hd = oracle_mod.lora_fwd(xd, d["w0"], d["a"], d["b"], alpha)
    np.testing.assert_array_equal(h, hd)
    y_base, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], zeros_b, alpha)
    y_lora, _ = oracle_mod.lora_fwd(xd, zeros_w, d["a"], d["b"], alpha)
    np.testing.assert_array_equal(y, y_base + y_lora)
    g = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, dropout=drop)
    gd = oracle_mod.lora_bwd(xd, d["w0"], d["a"], d["b"], d["dy"], alpha)
    np.testing.assert_array_equal(g["gh"], gd["gh"])
    np.testing.assert_array_equal(g["da"], gd["da"])
    np.testing.assert_array_equal(g["db"], gd["db"])
    dx_base = oracle_mod.lora_bwd(d["x"], d["w0"], zeros_a, d["b"], d["dy"], alpha)["dx"]
    dx_lora = oracle_mod.lora_bwd(d["x"], zeros_w, d["a"], d["b"], d["dy"], alpha)["dx"]
    dx_lora_d = oracle_mod.lora_bwd(d["x"], zeros_w, d["a"], d["b"], d["dy"], alpha, dropout=drop)["dx"]
    np.testing.assert_array_equal(dx_lora_d, 2.0 * M * dx_lora)
    np.testing.assert_array_equal(g["dx"], dx_base + dx_lora_d)


def test_dropout_finite_differences_exact(oracle_mod):
    """For a fixed mask L = <y, G> is linear in x, A and B: central differences
    with step 1 on ternary inputs (q = 2) are exact."""
    T, n, m, r = 6, 8, 8, 2
    alpha, drop = 4.0, (0.5, 11, 0)
    d = make_lora_inputs(T, n, m, r, seed=33, dist="ternary")
    g = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, dropout=drop)
    G = _f(d["dy"])

    def loss(x=None, a=None, b=None):
        y, _ = oracle_mod.lora_fwd(d["x"] if x is None else x, d["w0"], d["a"] if a is None else a,
                                   d["b"] if b is None else b, alpha, dropout=drop)
        return float(np.sum(y * G))

    def step(arr, idx, sign):
        v = _f(arr).astype(np.float32)
        v[idx] += sign
        return f32_to_bf16_bits(v)

    for t in range(T):
        for k in range(n):
            fd = (loss(x=step(d["x"], (t, k), 1.0)) - loss(x=step(d["x"], (t, k), -1.0))) / 2.0
            assert fd == g["dx"][t, k]
    for j in range(r):
        for k in range(n):
            fd = (loss(a=step(d["a"], (j, k), 1.0)) - loss(a=step(d["a"], (j, k), -1.0))) / 2.0
            assert fd == g["da"][j, k]
    for i in range(m):
        for j in range(r):
            fd = (loss(b=step(d["b"], (i, j), 1.0)) - loss(b=step(d["b"], (i, j), -1.0))) / 2.0
            assert fd == g["db"][i, j]

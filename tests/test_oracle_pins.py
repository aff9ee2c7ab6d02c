"""Pins for the fp64 CPU oracle (oracle/), against facts other than the oracle.

Each test names what fixes the expected value: a worked example derived from
the paper (tests/golden/), a special case that reduces to a library routine
(numpy BLAS matmul), an exact mathematical property of Eq. 1 (linearity ->
exact finite differences, Euler's identity for homogeneous maps, the merge
identity of Eq. 1 line 2), or a closed-form count.  Chosen so a dropped term,
a wrong sign/scale, or a transposed operand in the oracle fails at least one.
"""
import json
import os

import numpy as np
import pytest

from synth import bf16_bits_to_f64, f32_to_bf16_bits, make_lora_inputs, WORKLOADS

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")


def _bits(v):
    return f32_to_bf16_bits(np.asarray(v, np.float32))


def _f(bits):
    return bf16_bits_to_f64(bits)


# --------------------------------------------------------------------------- 1
def test_worked_example_exact(oracle_mod):
    """SPEC.md:324 merge example extended to fwd/bwd (SURVEY.md 8(c) pin 1)."""
    g = json.load(open(GOLDEN))
    inp, exp = g["inputs"], g["expected"]
    x, w0, a, b, dy = (_bits(inp[k]) for k in ("x", "w0", "a", "b", "dy"))
    y, h = oracle_mod.lora_fwd(x, w0, a, b, inp["alpha"])
    np.testing.assert_array_equal(h, exp["h"])
    np.testing.assert_array_equal(y, exp["y"])
    gr = oracle_mod.lora_bwd(x, w0, a, b, dy, inp["alpha"])
    np.testing.assert_array_equal(gr["gh"], exp["gh"])
    np.testing.assert_array_equal(gr["dx"], exp["dx"])
    np.testing.assert_array_equal(gr["da"], exp["da"])
    np.testing.assert_array_equal(gr["db"], exp["db"])
    np.testing.assert_array_equal(oracle_mod.lora_merge(w0, a, b, inp["alpha"]), exp["merged"])


def embed_worked_example(T=128, n=64, m=64, r=4):
    """The worked example zero-padded into an ABI-legal shape (d_in, d_out
    multiples of 8); used by the GPU bit-exact test too."""
    g = json.load(open(GOLDEN))["inputs"]
    X = np.zeros((T, n), np.float32); X[0, :2] = g["x"][0]
    W = np.zeros((m, n), np.float32); W[:2, :2] = g["w0"]
    A = np.zeros((r, n), np.float32); A[0, :2] = g["a"][0]
    B = np.zeros((m, r), np.float32); B[:2, 0] = [row[0] for row in g["b"]]
    G = np.zeros((T, m), np.float32); G[0, :2] = g["dy"][0]
    # alpha such that s = alpha / r = 1, as in the golden case
    return dict(x=_bits(X), w0=_bits(W), a=_bits(A), b=_bits(B), dy=_bits(G), alpha=float(r))


def test_worked_example_embedded(oracle_mod):
    e = embed_worked_example()
    g = json.load(open(GOLDEN))["expected"]
    y, h = oracle_mod.lora_fwd(e["x"], e["w0"], e["a"], e["b"], e["alpha"])
    exp_y = np.zeros_like(y); exp_y[0, :2] = g["y"][0]
    np.testing.assert_array_equal(y, exp_y)
    gr = oracle_mod.lora_bwd(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["alpha"])
    exp_dx = np.zeros_like(gr["dx"]); exp_dx[0, :2] = g["dx"][0]
    exp_da = np.zeros_like(gr["da"]); exp_da[0, :2] = g["da"][0]
    exp_db = np.zeros_like(gr["db"]); exp_db[:2, 0] = [v[0] for v in g["db"]]
    np.testing.assert_array_equal(gr["dx"], exp_dx)
    np.testing.assert_array_equal(gr["da"], exp_da)
    np.testing.assert_array_equal(gr["db"], exp_db)


# --------------------------------------------------------------------------- 2
def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("shape", [(37, 24, 40, 3), (64, 64, 64, 4)])
def test_b_zero_is_base_gemm(oracle_mod, shape):
    """Fresh adapter, B = 0: y = x W0^T, dX = G W0 (numpy BLAS),
    dA == 0 exactly, dB = s G^T (x A^T) (numpy)."""
    T, n, m, r = shape
    d = make_lora_inputs(T, n, m, r, seed=11, zero_b=True)
    alpha = 16.0
    X, W, A, G = (_f(d[k]) for k in ("x", "w0", "a", "dy"))
    y, h = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha)
    assert _rel(y, X @ W.T) < 1e-13
    gr = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
    assert np.all(gr["da"] == 0.0) and np.all(gr["gh"] == 0.0)
    assert _rel(gr["dx"], G @ W) < 1e-13
    assert _rel(gr["db"], (alpha / r) * G.T @ (X @ A.T)) < 1e-13
    assert _rel(h, X @ A.T) < 1e-13


def test_a_zero_and_w0_zero_special_cases(oracle_mod):
    """A = 0: y = x W0^T, dB == 0, dA = (s G B)^T x.  W0 = 0: y = s x A^T B^T,
    dX = s G B A -- all via numpy BLAS."""
    T, n, m, r = 33, 48, 40, 5
    alpha = 10.0
    s = alpha / r
    d = make_lora_inputs(T, n, m, r, seed=12)
    X, W, A, B, G = (_f(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    za = np.zeros_like(d["a"])
    y, _ = oracle_mod.lora_fwd(d["x"], d["w0"], za, d["b"], alpha)
    assert _rel(y, X @ W.T) < 1e-13
    gr = oracle_mod.lora_bwd(d["x"], d["w0"], za, d["b"], d["dy"], alpha)
    assert np.all(gr["db"] == 0.0)
    assert _rel(gr["da"], (s * G @ B).T @ X) < 1e-13
    assert _rel(gr["dx"], G @ W) < 1e-13
    zw = np.zeros_like(d["w0"])
    y, _ = oracle_mod.lora_fwd(d["x"], zw, d["a"], d["b"], alpha)
    assert _rel(y, s * (X @ A.T) @ B.T) < 1e-13
    gr = oracle_mod.lora_bwd(d["x"], zw, d["a"], d["b"], d["dy"], alpha)
    assert _rel(gr["dx"], s * (G @ B) @ A) < 1e-13


def test_bias_added_once(oracle_mod):
    """b0 of Eq. 1: with W0 = A = 0 the output is exactly b0."""
    T, n, m, r = 5, 16, 24, 2
    d = make_lora_inputs(T, n, m, r, seed=13, bias=True)
    z = np.zeros_like
    y, _ = oracle_mod.lora_fwd(d["x"], z(d["w0"]), z(d["a"]), d["b"], 16.0, bias=d["bias"])
    np.testing.assert_array_equal(y, np.broadcast_to(_f(d["bias"]), (T, m)))


# --------------------------------------------------------------------------- 3
def test_merge_equivalence(oracle_mod):
    """Eq. 1: W0 x + B A x == (W0 + B A) x, both for the
    output and for dX = G (W0 + s B A)."""
    T, n, m, r = 40, 56, 48, 6
    alpha = 12.0
    d = make_lora_inputs(T, n, m, r, seed=14)
    Wm = oracle_mod.lora_merge(d["w0"], d["a"], d["b"], alpha)
    X, G = _f(d["x"]), _f(d["dy"])
    y, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha)
    assert _rel(y, X @ Wm.T) < 1e-12
    gr = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
    assert _rel(gr["dx"], G @ Wm) < 1e-12


def test_merge_b_zero_is_identity(oracle_mod):
    """B = 0 -> merged == W0 exactly."""
    d = make_lora_inputs(4, 32, 24, 3, seed=15, zero_b=True)
    np.testing.assert_array_equal(oracle_mod.lora_merge(d["w0"], d["a"], d["b"], 16.0), _f(d["w0"]))


# --------------------------------------------------------------------------- 4
def _loss(oracle_mod, d, alpha, x=None, a=None, b=None):
    y, _ = oracle_mod.lora_fwd(d["x"] if x is None else x, d["w0"],
                               d["a"] if a is None else a, d["b"] if b is None else b, alpha)
    return float(np.sum(y * _f(d["dy"])))


def test_finite_differences_exact(oracle_mod):
    """L = <y, G> is linear in each of x, A, B separately, so a central
    difference with step 1 on small-integer (ternary) inputs is exact
    (SURVEY.md 8(c) pin 4).  Checks every entry of dA and dB
    and a sample of dX."""
    T, n, m, r = 6, 8, 8, 2
    alpha = 4.0
    d = make_lora_inputs(T, n, m, r, seed=16, dist="ternary")
    gr = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
    one = f32_to_bf16_bits(np.float32(1.0))

    def step(arr, idx, sign):
        v = _f(arr).astype(np.float32)
        v[idx] += sign
        return f32_to_bf16_bits(v)

    for j in range(r):
        for k in range(n):
            fd = (_loss(oracle_mod, d, alpha, a=step(d["a"], (j, k), 1.0)) -
                  _loss(oracle_mod, d, alpha, a=step(d["a"], (j, k), -1.0))) / 2.0
            assert fd == gr["da"][j, k]
    for i in range(m):
        for j in range(r):
            fd = (_loss(oracle_mod, d, alpha, b=step(d["b"], (i, j), 1.0)) -
                  _loss(oracle_mod, d, alpha, b=step(d["b"], (i, j), -1.0))) / 2.0
            assert fd == gr["db"][i, j]
    for (t, k) in [(0, 0), (1, 3), (5, 7), (3, 2)]:
        fd = (_loss(oracle_mod, d, alpha, x=step(d["x"], (t, k), 1.0)) -
              _loss(oracle_mod, d, alpha, x=step(d["x"], (t, k), -1.0))) / 2.0
        assert fd == gr["dx"][t, k]
    assert one == 0x3F80


def test_euler_identities(oracle_mod):
    """The LoRA term of <y, G> is linear (degree-1 homogeneous) in A and in B,
    and all of <y - b0, G> is linear in x, so by Euler's identity
        <dA, A> = <dB, B> = <y - y|_{B=0}, G>   and   <dX, x> = <y, G>.
    A transposed or mis-indexed gradient breaks these."""
    T, n, m, r = 29, 40, 32, 7
    alpha = 8.0
    d = make_lora_inputs(T, n, m, r, seed=17)
    y, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha)
    y0, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], np.zeros_like(d["b"]), alpha)
    G = _f(d["dy"])
    gr = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
    lora_l = np.sum((y - y0) * G)
    assert abs(np.sum(gr["da"] * _f(d["a"])) - lora_l) < 1e-10 * abs(lora_l)
    assert abs(np.sum(gr["db"] * _f(d["b"])) - lora_l) < 1e-10 * abs(lora_l)
    full_l = np.sum(y * G)
    assert abs(np.sum(gr["dx"] * _f(d["x"])) - full_l) < 1e-10 * abs(full_l)


def test_scale_law(oracle_mod):
    """s = alpha / r (Listing 3; R2): doubling alpha
    doubles y - y|_{B=0} exactly (powers of two are exact in fp64)."""
    T, n, m, r = 16, 24, 16, 4
    d = make_lora_inputs(T, n, m, r, seed=18)
    y1, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0)
    y2, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 32.0)
    y0, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], np.zeros_like(d["b"]), 16.0)
    np.testing.assert_allclose(y2 - y0, 2.0 * (y1 - y0), rtol=1e-12, atol=1e-12)
    # alpha == r -> s == 1 -> Eq. 1 verbatim: y = x W0^T + (x A^T) B^T
    X, W, A, B = (_f(d[k]) for k in ("x", "w0", "a", "b"))
    y4, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], float(r))
    assert _rel(y4, X @ W.T + (X @ A.T) @ B.T) < 1e-13


# --------------------------------------------------------------------------- 5
def test_row_subset_and_thread_independence(oracle_mod):
    """Rows are independent (each token row of y / dX depends only on that
    row): a row subset equals the same rows of the full result bitwise, and
    results do not depend on the OpenMP thread count."""
    T, n, m, r = 50, 32, 40, 3
    d = make_lora_inputs(T, n, m, r, seed=19)
    rows = np.array([49, 0, 17, 17, 3])
    yf, hf = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0)
    ys, hs = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0, rows=rows)
    np.testing.assert_array_equal(ys, yf[rows])
    np.testing.assert_array_equal(hs, hf[rows])
    gf = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
    gs = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, rows=rows)
    np.testing.assert_array_equal(gs["dx"], gf["dx"][rows])
    nt = oracle_mod.num_threads()
    oracle_mod.set_num_threads(1)
    try:
        g1 = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0)
        y1, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0)
    finally:
        oracle_mod.set_num_threads(nt)
    for k in ("dx", "da", "db", "gh"):
        np.testing.assert_array_equal(g1[k], gf[k])
    np.testing.assert_array_equal(y1, yf)


# --------------------------------------------------------------------------- 6
def test_tensor_parallel_partition_algebra(oracle_mod):
    """PAPER.md:122 sharding, read as Megatron column/row parallelism
    (R10/R11/R12): per-shard oracle results, combined by the
    partition rules (concatenate local outputs, sum partials in rank order),
    equal the unsharded oracle.  This pins the partition rules the TP layer
    implements."""
    T, n, m, r, N = 24, 32, 48, 4, 4
    alpha = 16.0
    d = make_lora_inputs(T, n, m, r, seed=20)
    y, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha)
    gr = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
    # column-parallel: W0, B split on m; A replicated
    ms = m // N
    ys, dxs, das, dbs = [], 0.0, 0.0, []
    for p in range(N):
        sl = slice(p * ms, (p + 1) * ms)
        yp, _ = oracle_mod.lora_fwd(d["x"], d["w0"][sl], d["a"], d["b"][sl], alpha)
        gp = oracle_mod.lora_bwd(d["x"], d["w0"][sl], d["a"], d["b"][sl],
                                 np.ascontiguousarray(d["dy"][:, sl]), alpha)
        ys.append(yp); dbs.append(gp["db"])
        dxs = dxs + gp["dx"]; das = das + gp["da"]
    assert _rel(np.concatenate(ys, 1), y) < 1e-13
    assert _rel(dxs, gr["dx"]) < 1e-13
    assert _rel(das, gr["da"]) < 1e-13          # sum, no 1/N (R12)
    assert _rel(np.concatenate(dbs, 0), gr["db"]) < 1e-13
    # row-parallel: W0, A split on n; B replicated.  Partial y and partial dB
    # (built from the local h) are summed; dX, dA are local.
    ns = n // N
    ysum, dbsum, dxs, das = 0.0, 0.0, [], []
    for p in range(N):
        sl = slice(p * ns, (p + 1) * ns)
        xp = np.ascontiguousarray(d["x"][:, sl])
        wp = np.ascontiguousarray(d["w0"][:, sl])
        ap = np.ascontiguousarray(d["a"][:, sl])
        yp, _ = oracle_mod.lora_fwd(xp, wp, ap, d["b"], alpha)
        gp = oracle_mod.lora_bwd(xp, wp, ap, d["b"], d["dy"], alpha)
        ysum = ysum + yp; dbsum = dbsum + gp["db"]
        dxs.append(gp["dx"]); das.append(gp["da"])
    assert _rel(ysum, y) < 1e-13
    assert _rel(dbsum, gr["db"]) < 1e-13
    assert _rel(np.concatenate(dxs, 1), gr["dx"]) < 1e-13
    assert _rel(np.concatenate(das, 1), gr["da"]) < 1e-13


# --------------------------------------------------------------------------- 7
def test_trainable_parameter_counts():
    """SPEC.md:341 closed form: trainable params = sum r (m + n).  Pins the
    workload shape table: 32 layers of 7B, r = 16."""
    def count(keys, r):
        wl = WORKLOADS["cfg3"]
        return sum(r * (l.m + l.n) for l in wl.linears if l.name in keys)
    assert 32 * count({"q", "v"}, 16) == 8_388_608
    assert 32 * count({"q", "k", "v", "o", "gate", "up", "down"}, 16) == 39_976_960


def test_bf16_rounding_is_rne():
    """The shared input generator rounds to nearest-even (ties to even)."""
    vals = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 65504.0], np.float32)
    bits = f32_to_bf16_bits(vals)
    np.testing.assert_array_equal(bf16_bits_to_f64(bits), [1.0, 1.0, 1.0 + 2 ** -6, -2.5, 65536.0])

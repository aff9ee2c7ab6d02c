"""Seeded fuzz of the grouped entry points (PAPER.md:115-120 Eq. 1, :111; Listing 3
LORA_DROPOUT): random ragged shapes, ranks 1..64, 1-4 members
sharing x, with and without LoRA dropout (kept mask or redrawn).  Every case
checks the grouped calls against the single calls -- y, h, dX bitwise, dA / dB
to fp32 re-association (include/lora.h: the dA/dB kernel's token split is
chosen per launch) -- and the single calls against the fp64 oracle within the
north-star tolerances."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_lora_inputs  # noqa: E402
from tests.gpu_util import TOL_GRAD, TOL_OUT, dev_bf16, host_f64, relF  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2403_11366_b200 as L
    L.lora_device_check()
    return L


def _cases(n_cases=14, seed=20260):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        T = int(rng.integers(1, 700))
        n = 8 * int(rng.integers(1, 80))
        G = int(rng.integers(1, 5))
        ms = [8 * int(rng.integers(1, 80)) for _ in range(G)]
        rs = [int(rng.choice([1, 3, 5, 8, 12, 16, 24, 33, 64])) for _ in range(G)]
        p = float(rng.choice([0.0, 0.0, 0.05, 0.3]))
        keep = bool(rng.integers(0, 2))
        out.append((i, T, n, tuple(ms), tuple(rs), p, keep))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}-T{c[1]}-n{c[2]}-G{len(c[3])}-p{c[5]}")
def test_grouped_fuzz(oracle_mod, L, case):
    i, T, n, ms, rs, p, keep = case
    alpha = 16.0
    base = make_lora_inputs(T, n, ms[0], rs[0], seed=30000 + i)
    x = dev_bf16(base["x"])
    ds, ts, drops = [], [], []
    for g, (m, r) in enumerate(zip(ms, rs)):
        d = make_lora_inputs(T, n, m, r, seed=30100 + 10 * i + g)
        d["x"] = base["x"]
        ds.append(d)
        ts.append({k: dev_bf16(d[k]) for k in ("w0", "a", "b", "dy")})
        if p > 0.0:
            dr = (p, 77 + g, 1000 * i + g)
            if keep:
                dr = dr + (L.dropout_keep_bits(T, n), torch.empty((T, n), dtype=torch.bfloat16, device="cuda"))
            drops.append(dr)
    dropouts = drops if p > 0.0 else None
    fo = L.lora_linear_fwd_grouped([(x, t["w0"], t["a"], t["b"], None) for t in ts], [alpha] * len(ts),
                                   dropouts=dropouts)
    go = L.lora_linear_bwd_grouped([(x, t["w0"], t["a"], t["b"], t["dy"], h) for t, (_, h) in zip(ts, fo)],
                                   [alpha] * len(ts), dropouts=dropouts)
    torch.cuda.synchronize()
    for g, (t, d) in enumerate(zip(ts, ds)):
        kw = {"dropout": drops[g]} if p > 0.0 else {}
        y1, h1 = L.lora_linear_fwd(x, t["w0"], t["a"], t["b"], alpha, **kw)
        dx1, da1, db1 = L.lora_linear_bwd(x, t["w0"], t["a"], t["b"], t["dy"], alpha, h_saved=h1, **kw)
        torch.cuda.synchronize()
        assert torch.equal(fo[g][0], y1) and torch.equal(fo[g][1], h1), (case, g)
        assert torch.equal(go[g][0], dx1), (case, g)
        for u, v in ((go[g][1], da1), (go[g][2], db1)):
            torch.testing.assert_close(u, v, rtol=1e-5, atol=1e-5 * float(v.abs().max()) + 1e-30)
        okw = {"dropout": drops[g][:3]} if p > 0.0 else {}
        yo, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, **okw)
        gor = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha, **okw)
        errs = (relF(host_f64(y1), yo), relF(host_f64(dx1), gor["dx"]), relF(host_f64(da1), gor["da"]),
                relF(host_f64(db1), gor["db"]))
        assert errs[0] <= TOL_OUT and errs[1] <= TOL_OUT, (case, g, errs)
        assert errs[2] <= TOL_GRAD and errs[3] <= TOL_GRAD, (case, g, errs)


def _single_cases(n_cases=12, seed=4242):
    rng = np.random.default_rng(seed)
    out = [(100, 1, 8, 8, 1), (101, 2, 8, 16, 64), (102, 129, 8, 4096, 16), (103, 3000, 4096, 8, 8)]
    for i in range(n_cases):
        out.append((i, int(rng.integers(1, 1500)), 8 * int(rng.integers(1, 200)), 8 * int(rng.integers(1, 200)),
                    int(rng.integers(1, 65))))
    return out


@pytest.mark.parametrize("case", _single_cases(), ids=lambda c: f"c{c[0]}-T{c[1]}-n{c[2]}-m{c[3]}-r{c[4]}")
def test_single_and_merge_fuzz(oracle_mod, L, case):
    """Single fwd / bwd (h saved and recomputed, dX skipped) and the merge at random
    and extreme shapes (T = 1, d = 8, r = 1 and 64, skinny and wide) against the
    oracle; the merge is >= 99.9% bit-equal to RNE(oracle) and within 1e-2."""
    from tests.gpu_util import rne_bf16_f64
    i, T, n, m, r = case
    d = make_lora_inputs(T, n, m, r, seed=40000 + i)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    alpha = 16.0
    y, h = L.lora_linear_fwd(x, w0, a, b, alpha)
    dx, da, db = L.lora_linear_bwd(x, w0, a, b, dy, alpha, h_saved=h)
    dx2, da2, db2 = L.lora_linear_bwd(x, w0, a, b, dy, alpha, h_saved=None, want_dx=False)
    wm = L.lora_merge(w0, a, b, alpha)
    torch.cuda.synchronize()
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
    assert relF(host_f64(y), yo) <= TOL_OUT and relF(host_f64(h), ho) <= 1e-4
    assert relF(host_f64(dx), go["dx"]) <= TOL_OUT
    for da_, db_ in ((da, db), (da2, db2)):
        assert relF(host_f64(da_), go["da"]) <= TOL_GRAD and relF(host_f64(db_), go["db"]) <= TOL_GRAD
    assert dx2 is None
    mo = oracle_mod.lora_merge(d["w0"], d["a"], d["b"], alpha)
    got = host_f64(wm)
    assert relF(got, mo) <= TOL_OUT
    assert np.sum(got != rne_bf16_f64(mo)) <= max(2, 0.001 * got.size)


@pytest.fixture(scope="module")
def comm(L):
    from paper_2403_11366_b200 import tp
    c = tp.LoraComm()
    yield c
    c.close()


def _tp_cases(n_cases=8, seed=777):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        out.append((i, int(rng.integers(1, 1300)), 8 * int(rng.integers(1, 100)), 8 * int(rng.integers(1, 100)),
                    int(rng.integers(1, 65)), str(rng.choice(["column", "row"])), str(rng.choice(["1", "3"])),
                    float(rng.choice([0.0, 0.05]))))
    return out


@pytest.mark.parametrize("case", _tp_cases(), ids=lambda c: f"c{c[0]}-T{c[1]}-{c[5]}-chunks{c[6]}-p{c[7]}")
def test_tp_n1_fuzz(L, comm, case, monkeypatch):
    """The tensor-parallel calls at N = 1 (real NCCL communicator) at random shapes,
    modes, forward token slicing and dropout: bitwise the single calls."""
    from paper_2403_11366_b200 import tp
    i, T, n, m, r, mode, chunks, p = case
    d = make_lora_inputs(T, n, m, r, seed=50000 + i)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    spec = tp.ShardSpec(tp.MODES[mode], 1, 0, n, m)
    drop = (p, 9 + i, 3 * i) if p > 0.0 else None
    kw = {"dropout": drop} if drop else {}
    y1, h1 = L.lora_linear_fwd(x, w0, a, b, 16.0, **kw)
    dx1, da1, db1 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h1, **kw)
    monkeypatch.setenv("LORA_TP_CHUNKS", chunks)
    y2, h2 = tp.tp_linear_fwd(comm, spec, x, w0, a, b, 16.0, dropout=drop)
    dx2, da2, db2 = tp.tp_linear_bwd(comm, spec, x, w0, a, b, dy, 16.0, h_saved=h2, dropout=drop)
    torch.cuda.synchronize()
    for u, v in ((y1, y2), (h1, h2), (dx1, dx2), (da1, da2), (db1, db2)):
        assert torch.equal(u, v), case


@pytest.mark.parametrize("case", _cases(n_cases=6, seed=99), ids=lambda c: f"g{c[0]}-T{c[1]}-n{c[2]}-G{len(c[3])}-p{c[5]}")
def test_grouped_graph_replay_fuzz(L, case):
    """The grouped forward + backward (dropout with kept mask / M.x when p > 0,
    accumulate into dA / dB) captured ONCE as a CUDA graph and replayed with new
    inputs written in place: bitwise the eager calls on those inputs (the
    self-cleaning sync words and the kept buffers carry no state across replays)."""
    i, T, n, ms, rs, p, _ = case
    alpha = 16.0
    gen = torch.Generator(device="cuda").manual_seed(1234 + i)
    x = torch.empty((T, n), dtype=torch.bfloat16, device="cuda")
    ts = []
    for m, r in zip(ms, rs):
        ts.append({"w0": torch.randn((m, n), device="cuda", generator=gen).bfloat16() / n ** 0.5,
                   "a": torch.randn((r, n), device="cuda", generator=gen).bfloat16() / n ** 0.5,
                   "b": torch.randn((m, r), device="cuda", generator=gen).bfloat16() / r ** 0.5,
                   "dy": torch.empty((T, m), dtype=torch.bfloat16, device="cuda")})
    drops = None
    if p > 0.0:
        drops = [(p, 5 + g, 7 * g, L.dropout_keep_bits(T, n), torch.empty((T, n), dtype=torch.bfloat16, device="cuda"))
                 for g in range(len(ts))]
    G = len(ts)
    ys = [(torch.empty((T, t["w0"].shape[0]), dtype=torch.bfloat16, device="cuda"),
           torch.empty((T, t["a"].shape[0]), dtype=torch.float32, device="cuda")) for t in ts]
    gs = [(torch.empty((T, n), dtype=torch.bfloat16, device="cuda"), torch.zeros_like(t["a"], dtype=torch.float32),
           torch.zeros_like(t["b"], dtype=torch.float32)) for t in ts]

    def fill(k):
        x.copy_(torch.randn((T, n), device="cuda", generator=gen))
        for t in ts:
            t["dy"].copy_(torch.randn(t["dy"].shape, device="cuda", generator=gen))

    def step(outs_f, outs_b, acc):
        L.lora_linear_fwd_grouped([(x, t["w0"], t["a"], t["b"], None) for t in ts], [alpha] * G, outs=outs_f,
                                  dropouts=drops)
        L.lora_linear_bwd_grouped([(x, t["w0"], t["a"], t["b"], t["dy"], h) for t, (_, h) in zip(ts, outs_f)],
                                  [alpha] * G, outs=outs_b, accumulate=acc, dropouts=drops)

    fill(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(ys, gs, True)   # (warm-up: workspaces allocated outside the capture)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step(ys, gs, True)
    for k in range(2):
        fill(k + 1)
        for _, da, db in gs:
            da.zero_()
            db.zero_()
        g.replay()
        torch.cuda.synchronize()
        ref_f = [(torch.empty_like(y), torch.empty_like(h)) for y, h in ys]
        ref_b = [(torch.empty_like(dx), torch.zeros_like(da), torch.zeros_like(db)) for dx, da, db in gs]
        step(ref_f, ref_b, True)
        torch.cuda.synchronize()
        for (y, h), (y1, h1) in zip(ys, ref_f):
            assert torch.equal(y, y1) and torch.equal(h, h1), (case, k)
        for (dx, da, db), (dx1, da1, db1) in zip(gs, ref_b):
            assert torch.equal(dx, dx1) and torch.equal(da, da1) and torch.equal(db, db1), (case, k)


def _drop_cases(n_cases=8, seed=31337):
    rng = np.random.default_rng(seed)
    return [(i, int(rng.integers(1, 900)), 8 * int(rng.integers(1, 120)), 8 * int(rng.integers(1, 120)),
             int(rng.integers(1, 65)), float(rng.choice([0.05, 0.2, 0.5])), bool(rng.integers(0, 2)),
             bool(rng.integers(0, 2)), bool(rng.integers(0, 2))) for i in range(n_cases)]


@pytest.mark.parametrize("case", _drop_cases(), ids=lambda c: f"d{c[0]}-T{c[1]}-r{c[4]}-p{c[5]}")
def test_dropout_single_paths_fuzz(oracle_mod, L, case):
    """Single dropout calls at random shapes and p, with the backward's h saved or
    recomputed, dX wanted or skipped, the mask kept or redrawn: vs the oracle, and
    every backward variant equal to the full one on what they share."""
    i, T, n, m, r, p, recompute, skip_dx, keep = case
    d = make_lora_inputs(T, n, m, r, seed=60000 + i)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    drop = (p, 40 + i, 5 * i)
    if keep:
        drop = drop + (L.dropout_keep_bits(T, n), torch.empty((T, n), dtype=torch.bfloat16, device="cuda"))
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=drop)
    dx, da, db = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dropout=drop)
    dx2, da2, db2 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=None if recompute else h,
                                      want_dx=not skip_dx, dropout=drop)
    torch.cuda.synchronize()
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], 16.0, dropout=drop[:3])
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, dropout=drop[:3])
    assert relF(host_f64(y), yo) <= TOL_OUT and relF(host_f64(h), ho) <= 1e-4, case
    assert relF(host_f64(dx), go["dx"]) <= TOL_OUT, case
    for da_, db_ in ((da, db), (da2, db2)):
        assert relF(host_f64(da_), go["da"]) <= TOL_GRAD and relF(host_f64(db_), go["db"]) <= TOL_GRAD, case
    if not skip_dx:
        assert relF(host_f64(dx2), go["dx"]) <= TOL_OUT, case
    else:
        assert dx2 is None

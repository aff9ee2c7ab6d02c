"""Parity of the exact path bench.py times ("parity-certify the
exact path that produces the numbers"): bench.StepRunner -- the grouped q+v
(cfg2) / layer-set (cfg3) calls on one shared x tensor per group, captured as
ONE CUDA graph and replayed -- against the fp64 oracle on the same seeded
inputs (PAPER.md:115-120 Eq. 1, :111).

cfg2 is checked on ALL 2048 token rows of y, h and dX and in full for dA, dB,
globally and per 32-row x 16-column block (a TMEM lane band of one output
tile), then replayed with NEW upstream gradients.  cfg3's groups (q/k/v,
gate/up) and single linears (o, down) are checked on the first 256, 128 random
and the last 32 rows."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import WORKLOADS, make_lora_inputs  # noqa: E402
from tests.gpu_util import TOL_GRAD, TOL_OUT, dev_bf16, host_f64, relF  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2403_11366_b200 as L
    L.lora_device_check()
    return torch.device("cuda", 0)


def block_relF_max(got, ref, br=32, bc=16):
    """max over (br x bc) blocks of ||got - ref||_F / ||ref||_F (ragged edges folded
    into the last block)."""
    T, N = ref.shape
    worst = 0.0
    for r0 in range(0, T, br):
        g = got[r0:r0 + br]
        f = ref[r0:r0 + br]
        nb = (N + bc - 1) // bc
        pad = nb * bc - N
        if pad:
            g = np.pad(g, ((0, 0), (0, pad)))
            f = np.pad(f, ((0, 0), (0, pad)))
        e = ((g - f) ** 2).reshape(g.shape[0], nb, bc).sum(axis=(0, 2))
        s = (f ** 2).reshape(f.shape[0], nb, bc).sum(axis=(0, 2))
        worst = max(worst, float(np.sqrt(np.max(e / np.maximum(s, 1e-300)))))
    return worst


def _check_linear(oracle_mod, e, d, rows=None, blocks=False, what=""):
    l = e["l"]
    yo, ho = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], l.alpha, rows=rows)
    go = oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], l.alpha, rows=rows)
    sel = slice(None) if rows is None else torch.as_tensor(rows, device=e["y"].device)
    got = {"y": host_f64(e["y"][sel]), "h": host_f64(e["h"][sel]), "dx": host_f64(e["dx"][sel]),
           "da": host_f64(e["da"]), "db": host_f64(e["db"])}
    errs = {"y": relF(got["y"], yo), "h": relF(got["h"], ho), "dx": relF(got["dx"], go["dx"]),
            "da": relF(got["da"], go["da"]), "db": relF(got["db"], go["db"])}
    if blocks:
        errs["y_block_max"] = block_relF_max(got["y"], yo)
        errs["dx_block_max"] = block_relF_max(got["dx"], go["dx"])
        errs["da_block_max"] = block_relF_max(got["da"], go["da"], br=1, bc=128)
        errs["db_block_max"] = block_relF_max(got["db"], go["db"], br=128, bc=l.r)
    print(what, l.name, {k: f"{v:.3e}" for k, v in errs.items()})
    assert errs["y"] <= TOL_OUT and errs["dx"] <= TOL_OUT, (what, l.name, errs)
    assert errs["da"] <= TOL_GRAD and errs["db"] <= TOL_GRAD, (what, l.name, errs)
    assert errs["h"] <= 1e-4, (what, l.name, errs)
    if blocks:
        assert errs["y_block_max"] <= TOL_OUT and errs["dx_block_max"] <= TOL_OUT, (what, l.name, errs)
        assert errs["da_block_max"] <= TOL_GRAD and errs["db_block_max"] <= TOL_GRAD, (what, l.name, errs)
    return errs


def test_cfg2_bench_step_graph_all_rows(oracle_mod, dev):
    """cfg2 exactly as timed: grouped q+v, shared x, one CUDA graph; every row."""
    import bench
    R = bench.StepRunner(WORKLOADS["cfg2"], dev)
    R.step()                       # warm-up outside capture (kernel attributes)
    torch.cuda.synchronize()
    graph, launches = R.capture(0)
    assert launches >= 3           # grouped K1, grouped K2, grouped K3
    for e in R.lin:                # poison the outputs: the replay must rewrite them
        for k in ("y", "dx", "da", "db", "h"):
            e[k].fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    for e, d in zip(R.lin, R.host):
        _check_linear(oracle_mod, e, d, blocks=True, what="cfg2 replay 1")
    y_first = [e["y"].clone() for e in R.lin]
    # replay with NEW upstream gradients (the graph reads dY through the same buffers)
    for i, e in enumerate(R.lin):
        l = e["l"]
        R.host[i] = dict(R.host[i], dy=make_lora_inputs(l.T, l.n, l.m, l.r, seed=7000 + i)["dy"])
        e["dy"].copy_(dev_bf16(R.host[i]["dy"]))
    graph.replay()
    torch.cuda.synchronize()
    for e, d, y0 in zip(R.lin, R.host, y_first):
        assert torch.equal(e["y"], y0)   # the forward does not depend on dY
        _check_linear(oracle_mod, e, d, blocks=True, what="cfg2 replay 2 (new dY)")


def test_cfg2_grouped_equals_single_calls_full_size(dev):
    """At the bench's full size the grouped, graph-replayed step equals the single
    eager calls bitwise for y, h, dX (same tiles, same k order) and to fp32
    re-association for dA, dB."""
    import bench

    import paper_2403_11366_b200 as L
    R = bench.StepRunner(WORKLOADS["cfg2"], dev)
    R.step()
    graph, _ = R.capture(0)
    graph.replay()
    torch.cuda.synchronize()
    for e in R.lin:
        y, h = L.lora_linear_fwd(e["x"], e["w0"], e["a"], e["b"], e["l"].alpha)
        dx, da, db = L.lora_linear_bwd(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["l"].alpha, h_saved=h)
        torch.cuda.synchronize()
        assert torch.equal(y, e["y"]) and torch.equal(h, e["h"]) and torch.equal(dx, e["dx"])
        torch.testing.assert_close(da, e["da"], rtol=1e-5, atol=1e-5 * float(da.abs().max()))
        torch.testing.assert_close(db, e["db"], rtol=1e-5, atol=1e-5 * float(db.abs().max()))


def test_cfg3_bench_step_graph_sampled_rows(oracle_mod, dev):
    """cfg3 (7B decoder-layer LoRA set, r 16, T 4096) exactly as timed: q/k/v and
    gate/up grouped on shared inputs, o and down single, one CUDA graph."""
    import bench
    R = bench.StepRunner(WORKLOADS["cfg3"], dev)
    R.step()
    torch.cuda.synchronize()
    graph, _ = R.capture(0)
    for e in R.lin:
        for k in ("y", "dx", "da", "db", "h"):
            e[k].fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    T = WORKLOADS["cfg3"].linears[0].T
    rng = np.random.default_rng(2403)
    rows = np.unique(np.concatenate([np.arange(256), rng.choice(T, 128, replace=False), np.arange(T - 32, T)]))
    for e, d in zip(R.lin, R.host):
        _check_linear(oracle_mod, e, d, rows=rows, what="cfg3")


def test_bench_parity_block(dev):
    """bench.StepRunner.parity() (the JSON line's `parity` block) reports pass on
    the timed outputs -- and fails on a corrupted output."""
    import bench
    R = bench.StepRunner(WORKLOADS["cfg2"], dev)
    R.step()
    p = R.parity()
    assert p["pass"], p
    R.lin[1]["dx"][1000:1032, 2048:2064] += 1.0   # one 32 x 16 block of one linear
    p = R.parity(rows_per_linear=np.arange(1000, 1032))
    assert not p["pass"], p

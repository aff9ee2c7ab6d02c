"""Tensor-parallel entry points on one B200 (N = 1): lora_tp_linear_fwd/bwd
through a real NCCL communicator owned by liblora.so must equal the
single-GPU calls bitwise (R13), in both COLUMN and ROW modes and
with the LoRA-gradient reduction inside or left to a bucketed all-reduce."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_lora_inputs  # noqa: E402
from tests.gpu_util import dev_bf16  # noqa: E402


@pytest.fixture(scope="module")
def comm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2403_11366_b200 import tp
    c = tp.LoraComm()
    yield c
    c.close()


@pytest.mark.parametrize("mode", ["column", "row"])
@pytest.mark.parametrize("accumulate", [False, True])
def test_tp_n1_equals_single_call(comm, mode, accumulate):
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    T, n, m, r = 384, 512, 640, 8
    d = make_lora_inputs(T, n, m, r, seed=61, bias=True)
    x, w0, a, b, dy, bias = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy", "bias"))
    spec = tp.ShardSpec(tp.MODES[mode], 1, 0, n, m)
    y1, h1 = L.lora_linear_fwd(x, w0, a, b, 16.0, bias=bias)
    y2, h2 = tp.tp_linear_fwd(comm, spec, x, w0, a, b, 16.0, bias=bias)
    da0 = torch.randn((r, n), device="cuda")
    db0 = torch.randn((m, r), device="cuda")
    dx1, da1, db1 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h1, da=da0.clone(), db=db0.clone(),
                                      accumulate=accumulate)
    dx2, da2, db2 = tp.tp_linear_bwd(comm, spec, x, w0, a, b, dy, 16.0, h_saved=h2, da=da0.clone(),
                                     db=db0.clone(), accumulate=accumulate)
    torch.cuda.synchronize()
    for u, v in ((y1, y2), (h1, h2), (dx1, dx2), (da1, da2), (db1, db2)):
        assert torch.equal(u, v)


def test_allreduce_n1_identity(comm):
    t = torch.randn(1000, device="cuda")
    ref = t.clone()
    comm.allreduce(t)
    torch.cuda.synchronize()
    assert torch.equal(t, ref)
    tb = torch.randn(1000, device="cuda").bfloat16()
    refb = tb.clone()
    comm.allreduce(tb)
    torch.cuda.synchronize()
    assert torch.equal(tb, refb)


def test_tp_column_group_sums_dx(comm, oracle_mod):
    """lora_tp_linear_bwd_column_group (q, k, v fused): the
    members' dX partials summed into the gradient w.r.t. the shared input, ONE
    all-reduce; dA, dB as the single calls.  Checked at N = 1 against the fp64
    oracle's sum of the members' dX."""
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    from tests.gpu_util import TOL_GRAD, TOL_OUT, host_f64, relF
    T, n = 512, 384
    base = make_lora_inputs(T, n, 8, 8, seed=70)
    x = dev_bf16(base["x"])
    specs, probs, refs, singles = [], [], [], []
    for i, (m, r) in enumerate([(256, 8), (136, 16), (192, 5)]):
        d = make_lora_inputs(T, n, m, r, seed=71 + i)
        d["x"] = base["x"]
        w0, a, b, dy = (dev_bf16(d[k]) for k in ("w0", "a", "b", "dy"))
        _, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
        specs.append(tp.ShardSpec(tp.COLUMN, 1, 0, n, m))
        probs.append((x, w0, a, b, dy, h))
        refs.append(oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0))
        singles.append(L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h))
    dx_sum, res = tp.tp_linear_bwd_column_group(comm, specs, probs, [16.0] * 3)
    torch.cuda.synchronize()
    assert relF(host_f64(dx_sum), sum(rf["dx"] for rf in refs)) <= TOL_OUT
    for (dx, da, db), (dx1, da1, db1), rf in zip(res, singles, refs):
        assert torch.equal(dx, dx1)                              # the members' own partials are kept
        assert relF(host_f64(da), rf["da"]) <= TOL_GRAD and relF(host_f64(db), rf["db"]) <= TOL_GRAD
        torch.testing.assert_close(da, da1, rtol=1e-5, atol=1e-5 * float(da1.abs().max()))


def test_tp_column_group_graph_replay(comm):
    """The column group forks its dX sum + all-reduce onto the communicator's side
    stream (overlapping the dA / dB kernel) and joins before the dA all-reduce:
    captured into a CUDA graph and replayed with new upstream gradients it must
    equal the eager call bitwise, every replay."""
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    T, n = 512, 384
    x = dev_bf16(make_lora_inputs(T, n, 8, 8, seed=80)["x"])
    specs, probs, dys, shapes = [], [], [], [(256, 8), (192, 16)]
    for i, (m, r) in enumerate(shapes):
        d = make_lora_inputs(T, n, m, r, seed=81 + i)
        w0, a, b = (dev_bf16(d[k]) for k in ("w0", "a", "b"))
        _, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
        dy = torch.empty((T, m), dtype=torch.bfloat16, device="cuda")
        dys.append(dy)
        specs.append(tp.ShardSpec(tp.COLUMN, 1, 0, n, m))
        probs.append((x, w0, a, b, dy, h))
    dx_sum = torch.empty((T, n), dtype=torch.bfloat16, device="cuda")
    outs = [(torch.empty((T, n), dtype=torch.bfloat16, device="cuda"), torch.empty((r, n), device="cuda"),
             torch.empty((m, r), device="cuda")) for (m, r) in shapes]
    ws = torch.empty(1 << 24, dtype=torch.uint8, device="cuda")

    def load(seed):
        for i, ((m, r), dy) in enumerate(zip(shapes, dys)):
            dy.copy_(dev_bf16(make_lora_inputs(T, n, m, r, seed=seed + i)["dy"]))
        torch.cuda.synchronize()

    s = torch.cuda.Stream()
    load(900)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        tp.tp_linear_bwd_column_group(comm, specs, probs, [16.0] * 2, dx_sum=dx_sum, outs=outs, workspace=ws,
                                      stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tp.tp_linear_bwd_column_group(comm, specs, probs, [16.0] * 2, dx_sum=dx_sum, outs=outs, workspace=ws,
                                      stream=s)
    for seed in (910, 920):
        load(seed)
        g.replay()
        torch.cuda.synchronize()
        got = [dx_sum.clone()] + [t.clone() for o in outs for t in o]
        ref_sum, ref = tp.tp_linear_bwd_column_group(comm, specs, probs, [16.0] * 2, workspace=ws)
        torch.cuda.synchronize()
        for u, v in zip(got, [ref_sum] + [t for o in ref for t in o]):
            assert torch.equal(u, v), f"replay {seed}"


@pytest.mark.parametrize("chunks", ["2", "3", "5"])
def test_tp_row_forward_token_slices(comm, chunks, monkeypatch):
    """ROW-parallel forward in token slices (slice i's all-reduce overlapping the GEMM
    of slice i + 1 on the communicator's side stream): y and h bitwise equal to the
    unsliced call, including a ragged last slice, eager and replayed as a CUDA graph."""
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    T, n, m, r = 1300, 256, 384, 8
    d = make_lora_inputs(T, n, m, r, seed=63, bias=True)
    x, w0, a, b, bias = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "bias"))
    spec = tp.ShardSpec(tp.ROW, 1, 0, n, m)
    y1, h1 = L.lora_linear_fwd(x, w0, a, b, 16.0, bias=bias)
    monkeypatch.setenv("LORA_TP_CHUNKS", chunks)
    y2, h2 = tp.tp_linear_fwd(comm, spec, x, w0, a, b, 16.0, bias=bias)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(h1, h2)
    # graph capture of the sliced fork / join
    y3 = torch.empty_like(y1)
    h3 = torch.empty_like(h1)
    ws = torch.empty(L.lora_linear_fwd_workspace_bytes(L.dims(T, n, m, r, 16.0)) + 256, dtype=torch.uint8,
                     device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            tp.tp_linear_fwd(comm, spec, x, w0, a, b, 16.0, bias=bias, y=y3, h_out=h3, workspace=ws, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    y3.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y1, y3) and torch.equal(h1, h3)


@pytest.mark.parametrize("mode", ["column", "row"])
@pytest.mark.parametrize("chunks", ["1", "3"])
def test_tp_dropout_n1_equals_single_call(comm, mode, chunks, monkeypatch):
    """lora_tp_linear_{fwd,bwd}_dropout at N = 1 (real NCCL communicator): bitwise
    the single-GPU dropout calls, also with the ROW forward in token slices (each
    slice draws its rows of the one mask; kept bits / M . x written per slice)."""
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    T, n, m, r = 700, 256, 384, 8
    d = make_lora_inputs(T, n, m, r, seed=67)
    x, w0, a, b, dy = (dev_bf16(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    spec = tp.ShardSpec(tp.MODES[mode], 1, 0, n, m)
    drop = (0.05, 11, 12)
    kb1, kb2 = L.dropout_keep_bits(T, n), L.dropout_keep_bits(T, n)
    mx1 = torch.empty((T, n), dtype=torch.bfloat16, device="cuda")
    mx2 = torch.empty_like(mx1)
    y1, h1 = L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=drop + (kb1, mx1))
    monkeypatch.setenv("LORA_TP_CHUNKS", chunks)
    y2, h2 = tp.tp_linear_fwd(comm, spec, x, w0, a, b, 16.0, dropout=drop + (kb2, mx2))
    dx1, da1, db1 = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h1, dropout=drop + (kb1, mx1))
    dx2, da2, db2 = tp.tp_linear_bwd(comm, spec, x, w0, a, b, dy, 16.0, h_saved=h2, dropout=drop + (kb2, mx2))
    torch.cuda.synchronize()
    for u, v in ((y1, y2), (h1, h2), (kb1, kb2), (mx1, mx2), (dx1, dx2), (da1, da2), (db1, db2)):
        assert torch.equal(u, v)


def test_tp_column_group_dropout(comm, oracle_mod):
    """lora_tp_linear_bwd_column_group_dropout at N = 1: the members' dX / dA / dB
    bitwise the grouped single-GPU dropout backward (each member its own mask, the
    forward's h), dx_sum == the oracle's sum of the members' dropout dX."""
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    from tests.gpu_util import TOL_OUT, host_f64, relF
    T, n = 384, 256
    base = make_lora_inputs(T, n, 8, 8, seed=90)
    x = dev_bf16(base["x"])
    specs, probs, drops, refs = [], [], [], []
    members = [(256, 8), (128, 8)]
    ts = []
    for i, (m, r) in enumerate(members):
        d = make_lora_inputs(T, n, m, r, seed=91 + i)
        d["x"] = base["x"]
        ts.append({k: dev_bf16(d[k]) for k in ("w0", "a", "b", "dy")})
        drops.append((0.05, 200 + i, 3 * i))
        specs.append(tp.ShardSpec(tp.COLUMN, 1, 0, n, m))
        refs.append(oracle_mod.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], 16.0, dropout=drops[-1]))
    fo = L.lora_linear_fwd_grouped([(x, t["w0"], t["a"], t["b"], None) for t in ts], [16.0] * 2, dropouts=drops)
    probs = [(x, t["w0"], t["a"], t["b"], t["dy"], h) for t, (_, h) in zip(ts, fo)]
    g1 = L.lora_linear_bwd_grouped(probs, [16.0] * 2, dropouts=drops)
    dx_sum, res = tp.tp_linear_bwd_column_group(comm, specs, probs, [16.0] * 2, dropouts=drops)
    torch.cuda.synchronize()
    for (dx, da, db), (dx1, da1, db1) in zip(res, g1):
        assert torch.equal(dx, dx1) and torch.equal(da, da1) and torch.equal(db, db1)
    assert relF(host_f64(dx_sum), sum(rf["dx"] for rf in refs)) <= TOL_OUT

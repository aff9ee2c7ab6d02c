"""Comm-fused epilogues over peer memory (lora_symm.cu) on one
B200: N "virtual ranks" of this process (lora_symm_connect_local), each with its
own symmetric buffer and stream, run the real protocol -- every rank's fused
GEMM publishes its 128-row output units, each rank's reducer sums the units it
owns over ranks (and group members) and stores the result into every rank's
buffer.  Checked against the UNSHARDED fp64 oracle (SURVEY.md 8(c) pin 8), all
ranks bitwise identical, repeat runs bitwise equal (R13), N = 1 equal
to the single-GPU call bitwise.  A two-process test maps the buffers with CUDA
IPC (the multi-GPU path) on the same device."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_lora_inputs  # noqa: E402
from tests.gpu_util import TOL_GRAD, TOL_OUT, dev_bf16, host_f64, relF  # noqa: E402


def _row_fwd(bufs, d, alpha, N, n, m, streams, h_outs=None):
    from paper_2403_11366_b200 import tp
    inputs = []
    for r in range(N):   # (all uploads first: nothing may synchronize between the ranks' calls)
        spec = tp.ShardSpec(tp.ROW, N, r, n, m)
        w0, a, b, bias = tp.shard_params(spec, d["w0"], d["a"], d["b"], d["bias"])
        inputs.append((spec, dev_bf16(tp.shard_input(spec, d["x"])), dev_bf16(w0), dev_bf16(a), dev_bf16(b),
                       dev_bf16(bias)))
    torch.cuda.synchronize()
    ys = []
    for r in range(N):
        spec, x, w0, a, b, bias = inputs[r]
        with torch.cuda.stream(streams[r]):
            y, _ = tp.tp_linear_fwd_fused(bufs[r], spec, x, w0, a, b, alpha, bias=bias, stream=streams[r])
        ys.append(y)
    torch.cuda.synchronize()
    return [y.clone() for y in ys]


@pytest.mark.parametrize("N,T,n,m,r", [(1, 384, 512, 768, 8), (2, 384, 512, 768, 8), (4, 300, 1024, 520, 16),
                                       (2, 1024, 2048, 2048, 8), (8, 256, 1024, 256, 4)])
def test_row_fwd_fused_virtual_ranks(oracle_mod, N, T, n, m, r):
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    alpha = 16.0
    d = make_lora_inputs(T, n, m, r, seed=700 + N, bias=True)
    yo, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, bias=d["bias"])
    bufs = tp.SymmBuffer.local_group(N, 2 * T * m * 2 + 4096)
    streams = [torch.cuda.Stream() for _ in range(N)]
    try:
        ys = _row_fwd(bufs, d, alpha, N, n, m, streams)
        for y in ys[1:]:
            assert torch.equal(y, ys[0])          # every rank holds the same reduced y
        assert relF(host_f64(ys[0]), yo) <= TOL_OUT
        ys2 = _row_fwd(bufs, d, alpha, N, n, m, streams)
        assert torch.equal(ys2[0], ys[0])         # repeat run: bitwise (fixed summation order)
        if N == 1:
            y1, _ = L.lora_linear_fwd(dev_bf16(d["x"]), dev_bf16(d["w0"]), dev_bf16(d["a"]), dev_bf16(d["b"]),
                                      alpha, bias=dev_bf16(d["bias"]))
            torch.cuda.synchronize()
            assert torch.equal(ys[0], y1)
    finally:
        for b in bufs:
            b.close()


def _col_group_bwd(bufs, d_list, alpha, N, n, ms, streams):
    from paper_2403_11366_b200 import tp
    import paper_2403_11366_b200 as L
    # every rank's inputs (and its forward h) first: the virtual ranks' fused calls are
    # then enqueued back to back -- rank 0's reducer waits for rank 1's dX kernel, so
    # nothing may synchronize the device between them
    inputs = []
    for r in range(N):
        specs, probs = [], []
        x = dev_bf16(d_list[0]["x"])
        for g, d in enumerate(d_list):
            spec = tp.ShardSpec(tp.COLUMN, N, r, n, ms[g])
            w0, a, b, _ = tp.shard_params(spec, d["w0"], d["a"], d["b"])
            dy = dev_bf16(tp.shard_output_grad(spec, d["dy"]))
            w0, a, b = dev_bf16(w0), dev_bf16(a), dev_bf16(b)
            _, h = L.lora_linear_fwd(x, w0, a, b, alpha)
            specs.append(spec)
            probs.append((x, w0, a, b, dy, h))
        inputs.append((specs, probs))
    torch.cuda.synchronize()
    outs = []
    for r in range(N):
        specs, probs = inputs[r]
        with torch.cuda.stream(streams[r]):
            dxs, grads = tp.tp_linear_bwd_column_group_fused(bufs[r], specs, probs, [alpha] * len(d_list),
                                                             stream=streams[r])
        outs.append((dxs, grads))
    torch.cuda.synchronize()
    return [(dxs.clone(), [(da.clone(), db.clone()) for da, db in g]) for dxs, g in outs]


@pytest.mark.parametrize("N,T,n,ms,r", [(1, 384, 512, (512, 256, 256), 8), (2, 384, 512, (512, 256, 256), 8),
                                        (4, 520, 1024, (1024, 512), 16)])
def test_column_group_bwd_fused_virtual_ranks(oracle_mod, N, T, n, ms, r):
    from paper_2403_11366_b200 import tp
    alpha = 16.0
    base = make_lora_inputs(T, n, ms[0], r, seed=800 + N)
    d_list = []
    for g, m in enumerate(ms):
        dg = make_lora_inputs(T, n, m, r, seed=810 + 10 * N + g)
        dg["x"] = base["x"]
        d_list.append(dg)
    ref = [oracle_mod.lora_bwd(dg["x"], dg["w0"], dg["a"], dg["b"], dg["dy"], alpha) for dg in d_list]
    dx_ref = sum(o["dx"] for o in ref)
    G = len(ms)
    bufs = tp.SymmBuffer.local_group(N, (G + 1) * T * n * 2 + 4096)
    streams = [torch.cuda.Stream() for _ in range(N)]
    try:
        res = _col_group_bwd(bufs, d_list, alpha, N, n, ms, streams)
        for dxs, _ in res[1:]:
            assert torch.equal(dxs, res[0][0])
        assert relF(host_f64(res[0][0]), dx_ref) <= TOL_OUT
        for g, m in enumerate(ms):
            da = sum(host_f64(res[rk][1][g][0]) for rk in range(N))     # dA: partial per rank (R12: SUM)
            assert relF(da, ref[g]["da"]) <= TOL_GRAD
            db = np.concatenate([host_f64(res[rk][1][g][1]) for rk in range(N)], axis=0)   # dB: local rows
            assert relF(db, ref[g]["db"]) <= TOL_GRAD
        res2 = _col_group_bwd(bufs, d_list, alpha, N, n, ms, streams)
        assert torch.equal(res2[0][0], res[0][0])
    finally:
        for b in bufs:
            b.close()


def test_symm_region_validation():
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    bufs = tp.SymmBuffer.local_group(2, 1 << 20)
    try:
        spec = tp.ShardSpec(tp.ROW, 2, 0, 256, 256)
        x = torch.zeros((256, 128), dtype=torch.bfloat16, device="cuda")
        w0 = torch.zeros((256, 128), dtype=torch.bfloat16, device="cuda")
        a = torch.zeros((8, 128), dtype=torch.bfloat16, device="cuda")
        b = torch.zeros((256, 8), dtype=torch.bfloat16, device="cuda")
        with pytest.raises(L.LoraError, match="exceeds the symmetric data region"):
            tp.tp_linear_fwd_fused(bufs[0], spec, x, w0, a, b, 16.0, part_offset=(1 << 20) - 4096)
        with pytest.raises(L.LoraError, match="overlap"):
            tp.tp_linear_fwd_fused(bufs[0], spec, x, w0, a, b, 16.0, part_offset=0, y_offset=256)
    finally:
        for b_ in bufs:
            b_.close()


# ------------------------------------------------------------- CUDA IPC, 2 processes
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)   # both processes on the one GPU: IPC maps the peer's buffer
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import oracle
        from paper_2403_11366_b200 import tp
        T, n, m, r, alpha = 256, 512, 512, 8, 16.0
        d = make_lora_inputs(T, n, m, r, seed=901, bias=True)
        buf = tp.SymmBuffer(2 * T * m * 2 + 4096)
        spec = tp.ShardSpec(tp.ROW, world, rank, n, m)
        w0, a, b, bias = tp.shard_params(spec, d["w0"], d["a"], d["b"], d["bias"])
        y, _ = tp.tp_linear_fwd_fused(buf, spec, dev_bf16(tp.shard_input(spec, d["x"])), dev_bf16(w0),
                                      dev_bf16(a), dev_bf16(b), alpha, bias=dev_bf16(bias))
        torch.cuda.synchronize()
        yo, _ = oracle.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, bias=d["bias"])
        err = relF(host_f64(y), yo)
        digest = int(y.view(torch.int16).to(torch.int64).sum().item())
        dist.barrier()
        buf.close()
        q.put((rank, err, digest, None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, repr(e)))


def test_row_fwd_fused_ipc_two_processes():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, err, digest, exc in res:
        assert exc is None, exc
        assert err <= TOL_OUT
    assert res[0][2] == res[1][2]   # both processes hold the same reduced y


def _ipc_col_worker(rank, world, port, r, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import oracle
        import paper_2403_11366_b200 as L
        from paper_2403_11366_b200 import tp
        T, n, ms, alpha = 256, 512, (512, 256), 16.0
        base = make_lora_inputs(T, n, ms[0], r, seed=950)
        ds = []
        for g, m in enumerate(ms):
            dg = make_lora_inputs(T, n, m, r, seed=951 + g)
            dg["x"] = base["x"]
            ds.append(dg)
        x = dev_bf16(base["x"])
        specs, probs = [], []
        for g, (dg, m) in enumerate(zip(ds, ms)):
            spec = tp.ShardSpec(tp.COLUMN, world, rank, n, m)
            w0, a, b, _ = tp.shard_params(spec, dg["w0"], dg["a"], dg["b"])
            w0, a, b = dev_bf16(w0), dev_bf16(a), dev_bf16(b)
            _, h = L.lora_linear_fwd(x, w0, a, b, alpha)
            specs.append(spec)
            probs.append((x, w0, a, b, dev_bf16(tp.shard_output_grad(spec, dg["dy"])), h))
        buf = tp.SymmBuffer(3 * T * n * 2 + 4096)
        torch.cuda.synchronize()
        dx, _ = tp.tp_linear_bwd_column_group_fused(buf, specs, probs, [alpha] * 2)
        torch.cuda.synchronize()
        ref = sum(oracle.lora_bwd(dg["x"], dg["w0"], dg["a"], dg["b"], dg["dy"], alpha)["dx"] for dg in ds)
        err = relF(host_f64(dx), ref)
        digest = int(dx.view(torch.int16).to(torch.int64).sum().item())
        placement = buf.last_placement
        dist.barrier()
        buf.close()
        q.put((rank, err, digest, placement, None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, None, repr(e)))


@pytest.mark.parametrize("r", [8, 32])
def test_column_group_fused_ipc_two_processes(r):
    """The CUDA IPC path of the fused column-group backward (one rank per process,
    like one per GPU): r = 8 (the reducer fits next to the dX kernel: co-resident)
    and r = 32 (a 226-register dX kernel leaves no room: the reducer runs after it)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_col_worker, args=(rk, 2, port, r, q)) for rk in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, err, digest, placement, exc in res:
        assert exc is None, exc
        assert err <= TOL_OUT
    assert res[0][2] == res[1][2]
    assert res[0][3] == ("coresident" if r == 8 else "after_gemm"), res[0][3]


def _symm_cases(n_cases=6, seed=8080):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        N = int(rng.choice([2, 4]))
        out.append((i, N, int(rng.integers(1, 700)), 8 * N * int(rng.integers(1, 40)),
                    8 * N * int(rng.integers(1, 40)), int(rng.choice([4, 8, 16, 24]))))
    return out


@pytest.mark.parametrize("case", _symm_cases(), ids=lambda c: f"s{c[0]}-N{c[1]}-T{c[2]}")
def test_symm_fuzz(oracle_mod, case):
    """Seeded random shapes for both comm-fused protocols at 2 / 4 virtual ranks:
    the ROW forward's reduced y and the COLUMN-group backward's reduced dX (two
    members) against the UNSHARDED oracle, ranks bitwise identical."""
    from paper_2403_11366_b200 import tp
    i, N, T, n, m, r = case
    alpha = 16.0
    d = make_lora_inputs(T, n, m, r, seed=9000 + i, bias=True)
    yo, _ = oracle_mod.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, bias=d["bias"])
    bufs = tp.SymmBuffer.local_group(N, 2 * T * m * 2 + 4096)
    streams = [torch.cuda.Stream() for _ in range(N)]
    try:
        ys = _row_fwd(bufs, d, alpha, N, n, m, streams)
        for y in ys[1:]:
            assert torch.equal(y, ys[0])
        assert relF(host_f64(ys[0]), yo) <= TOL_OUT
    finally:
        for b in bufs:
            b.close()
    ms = (m, 8 * N * (1 + i))
    d_list = []
    for g, mm in enumerate(ms):
        dg = make_lora_inputs(T, n, mm, r, seed=9100 + 10 * i + g)
        dg["x"] = d["x"]
        d_list.append(dg)
    ref = [oracle_mod.lora_bwd(dg["x"], dg["w0"], dg["a"], dg["b"], dg["dy"], alpha) for dg in d_list]
    bufs = tp.SymmBuffer.local_group(N, (len(ms) + 1) * T * n * 2 + 4096)
    try:
        res = _col_group_bwd(bufs, d_list, alpha, N, n, ms, streams)
        for dxs, _ in res[1:]:
            assert torch.equal(dxs, res[0][0])
        assert relF(host_f64(res[0][0]), sum(o["dx"] for o in ref)) <= TOL_OUT
    finally:
        for b in bufs:
            b.close()

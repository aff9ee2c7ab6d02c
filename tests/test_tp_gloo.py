"""World-size-2 and -4 CPU (gloo) tests of the tensor-parallel host logic
(paper_2403_11366_b200/tp.py): each rank takes its shard with the product's
sharding functions, computes its local results (with the fp64 oracle standing
in for the per-rank kernels, CPU only), and the partial results that
`partial_outputs` names are SUM-all-reduced over gloo.  The combined result
must equal the unsharded oracle (PAPER.md:122 read as column/row parallelism,
DESIGN.md R10-R12)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode_name, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2403_11366_b200 import tp
        from synth import make_lora_inputs
        T, n, m, r, alpha = 24, 64, 96, 4, 16.0   # shards of 16 / 32 and 24 / 48 columns
        d = make_lora_inputs(T, n, m, r, seed=77, bias=True)
        spec = tp.ShardSpec(tp.MODES[mode_name], world, rank, n, m)
        w0, a, b, bias = tp.shard_params(spec, d["w0"], d["a"], d["b"], d["bias"])
        x = np.ascontiguousarray(tp.shard_input(spec, d["x"]))
        dy = np.ascontiguousarray(tp.shard_output_grad(spec, d["dy"]))
        w0, a, b = (np.ascontiguousarray(t) for t in (w0, a, b))
        # row mode: bias only on rank 0 (lora_tp_linear_fwd does the same)
        if spec.mode == tp.ROW and rank != 0:
            bias = None
        y, _ = oracle.lora_fwd(x, w0, a, b, alpha, bias=np.ascontiguousarray(bias) if bias is not None else None)
        g = oracle.lora_bwd(x, w0, a, b, dy, alpha)
        out = {"y": y, "dx": g["dx"], "da": g["da"], "db": g["db"]}
        for k, partial in tp.partial_outputs(spec).items():
            if partial:
                t = torch.from_numpy(out[k])
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
                out[k] = t.numpy()
        # gather the local (sharded) outputs to rank 0
        gathered = {}
        for k in out:
            objs = [None] * world
            dist.all_gather_object(objs, out[k])
            gathered[k] = objs
        if rank == 0:
            yo, _ = oracle.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, bias=d["bias"])
            go = oracle.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
            ref = {"y": yo, "dx": go["dx"], "da": go["da"], "db": go["db"]}
            axis = {"column": {"y": 1, "db": 0}, "row": {"dx": 1, "da": 1}}[mode_name]
            errs = {}
            for k in ref:
                if tp.partial_outputs(spec)[k]:
                    full = gathered[k][0]
                    assert all(np.array_equal(full, o) for o in gathered[k]), k  # replicated after reduce
                elif k in axis:
                    full = np.concatenate(gathered[k], axis=axis[k])
                else:
                    full = gathered[k][0]
                errs[k] = float(np.linalg.norm(full - ref[k]) / np.linalg.norm(ref[k]))
            q.put(("ok", errs))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e)))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["column", "row"])
def test_tp_gloo_matches_unsharded(mode, world, oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = []
    while not q.empty():
        res.append(q.get())
    assert res and all(s == "ok" for s, _ in res), res
    errs = [e for s, e in res if s == "ok"][0]
    assert all(v < 1e-12 for v in errs.values()), errs


def test_shard_spec_divisibility_errors():
    from paper_2403_11366_b200 import tp
    with pytest.raises(ValueError, match="d_out = 11008 is not divisible by N = 3"):
        tp.ShardSpec(tp.COLUMN, 3, 0, 4096, 11008)
    with pytest.raises(ValueError, match="shard of d_in = 12"):
        tp.ShardSpec(tp.ROW, 2, 0, 24, 4096)              # 12-column shards break 16-byte TMA rows
    with pytest.raises(ValueError, match="bad rank"):
        tp.ShardSpec(tp.ROW, 2, 2, 64, 64)
    spec = tp.ShardSpec(tp.ROW, 8, 3, 11008, 4096)
    assert spec.local_n == 1376 and spec.local_m == 4096 and spec.slice() == slice(4128, 5504)
    spec = tp.ShardSpec(tp.COLUMN, 8, 7, 4096, 11008)
    assert spec.local_m == 1376 and spec.slice() == slice(9632, 11008)
    assert tp.partial_outputs(spec) == {"y": False, "dx": True, "da": True, "db": False}

"""Tensor-parallel LoRA linear on >= 2 GPUs (R10-R13):
one process per GPU, the NCCL communicator owned by liblora.so, the gathered
sharded results against the UNSHARDED fp64 oracle (SURVEY.md 8(c) pin 8) for
COLUMN, ROW and the column group, repeat runs bitwise equal at fixed N, and
gradient accumulation with the LoRA-gradient reduction (the
accumulate + reduce path).  Skipped where fewer than 2 GPUs are visible (the
round's GPU boxes have one; the 1-rank path runs in test_gpu_tp.py)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    try:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
        import oracle
        import paper_2403_11366_b200 as L
        from paper_2403_11366_b200 import tp
        from synth import make_lora_inputs
        from tests.gpu_util import TOL_GRAD, TOL_OUT, dev_bf16, host_f64, relF
        comm = tp.LoraComm()
        T, n, m, r, alpha = 384, 512, 768, 8, 16.0
        d = make_lora_inputs(T, n, m, r, seed=1234, bias=True)
        yo, _ = oracle.lora_fwd(d["x"], d["w0"], d["a"], d["b"], alpha, bias=d["bias"])
        go = oracle.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], alpha)
        errs = {}
        for mode_name, mode in tp.MODES.items():
            spec = tp.ShardSpec(mode, world, rank, n, m)
            w0, a, b, bias = tp.shard_params(spec, d["w0"], d["a"], d["b"], d["bias"])
            x = dev_bf16(tp.shard_input(spec, d["x"]))
            dy = dev_bf16(tp.shard_output_grad(spec, d["dy"]))
            w0, a, b, bias = dev_bf16(w0), dev_bf16(a), dev_bf16(b), dev_bf16(bias)
            runs = []
            for _ in range(2):
                y, h = tp.tp_linear_fwd(comm, spec, x, w0, a, b, alpha, bias=bias)
                dx, da, db = tp.tp_linear_bwd(comm, spec, x, w0, a, b, dy, alpha, h_saved=h)
                torch.cuda.synchronize()
                runs.append([t.clone() for t in (y, dx, da, db)])
            for u, v in zip(*runs):
                assert torch.equal(u, v), f"{mode_name}: repeat run differs"
            y, dx, da, db = runs[0]
            sl = spec.slice()
            if mode == tp.COLUMN:   # y local columns; dX, dA reduced (full); dB local rows
                ref = {"y": yo[:, sl], "dx": go["dx"], "da": go["da"], "db": go["db"][sl]}
            else:                   # y reduced (full); dX, dA local columns; dB reduced (full)
                ref = {"y": yo, "dx": go["dx"][:, sl], "da": go["da"][:, sl], "db": go["db"]}
            got = {"y": host_f64(y), "dx": host_f64(dx), "da": host_f64(da), "db": host_f64(db)}
            e = {k: relF(got[k], ref[k]) for k in ref}
            errs[mode_name] = e
            assert e["y"] <= TOL_OUT and e["dx"] <= TOL_OUT, (mode_name, e)
            assert e["da"] <= TOL_GRAD and e["db"] <= TOL_GRAD, (mode_name, e)
            # accumulate + reduce_lora_grads: grad = old + reduced new, for BOTH factors
            da0 = torch.full_like(da, 0.5)
            db0 = torch.full_like(db, -0.25)
            _, da2, db2 = tp.tp_linear_bwd(comm, spec, x, w0, a, b, dy, alpha, h_saved=h, da=da0.clone(),
                                           db=db0.clone(), accumulate=True)
            torch.cuda.synchronize()
            assert relF(host_f64(da2) - 0.5, ref["da"]) <= TOL_GRAD, mode_name
            assert relF(host_f64(db2) + 0.25, ref["db"]) <= TOL_GRAD, mode_name
        # column group: q/k/v-style members sharing x, dX partials summed, ONE all-reduce
        specs, probs, refs = [], [], []
        xd = dev_bf16(d["x"])
        for i, (mm, rr) in enumerate([(256, 8), (512, 16)]):
            di = make_lora_inputs(T, n, mm, rr, seed=1300 + i)
            di["x"] = d["x"]
            spec = tp.ShardSpec(tp.COLUMN, world, rank, n, mm)
            w0, a, b, _ = tp.shard_params(spec, di["w0"], di["a"], di["b"])
            w0, a, b = dev_bf16(w0), dev_bf16(a), dev_bf16(b)
            dy = dev_bf16(tp.shard_output_grad(spec, di["dy"]))
            _, h = L.lora_linear_fwd(xd, w0, a, b, alpha)
            specs.append(spec)
            probs.append((xd, w0, a, b, dy, h))
            refs.append((spec, oracle.lora_bwd(di["x"], di["w0"], di["a"], di["b"], di["dy"], alpha)))
        dx_sum, res = tp.tp_linear_bwd_column_group(comm, specs, probs, [alpha] * 2)
        torch.cuda.synchronize()
        assert relF(host_f64(dx_sum), sum(rf["dx"] for _, rf in refs)) <= TOL_OUT
        for (spec, rf), (_, da, db) in zip(refs, res):
            assert relF(host_f64(da), rf["da"]) <= TOL_GRAD
            assert relF(host_f64(db), rf["db"][spec.slice()]) <= TOL_GRAD
        comm.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", errs))
    except Exception as ex:  # report to the parent instead of hanging it
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
        raise


def test_tp_world2_vs_unsharded_oracle():
    if not torch.cuda.is_available() or torch.cuda.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs (this box has {torch.cuda.device_count()})")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, WORLD, port, q)) for rk in range(WORLD)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    bad = [r for r in results if r[1] != "ok"]
    assert not bad, bad
    print(np.array(results, dtype=object))

#!/usr/bin/env python
"""Benchmark of the LoRA-linear hot path (JORA, arXiv 2403.11366) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg3|cfg4|cfg5]

Metric (BASELINE.json): LoRA-linear fwd+bwd TFLOP/s (% of bf16 peak) and
tokens/s.  One step = forward + backward of every LoRA linear of the workload
(cfg2 = Llama-2-7B q and v projections, 4096 x 4096, r = 8, alpha = 16,
batch 1 x seq 2048) on synthetic seeded bf16 data with inputs resident in HBM.
FLOPs are algorithmic: 4 T m n + 6 T r (m + n) per linear (no dW0, no padding).
At N > 1 the same global problem is tensor-sharded (column
parallel q, v) over N processes launched by torchrun: strong scaling, NCCL
all-reduces of dX and the LoRA-gradient bucket inside the step.

Prints ONE JSON line on rank 0.  `--impl reference` times the fp64 CPU oracle
(oracle/, the parity reference) on a bounded token sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from synth import WORKLOADS, algorithmic_flops, make_lora_inputs  # noqa: E402

FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def workload_flops(wl, T=None):
    return sum(algorithmic_flops(T or l.T, l.n, l.m, l.r) for l in wl.linears)


def gpu_local_cpus(dev_index):
    """CPUs on the same NUMA node as GPU `dev_index` (from sysfs), or None."""
    try:
        import torch
        bus = torch.cuda.get_device_properties(dev_index).pci_bus_id.lower()
        dom, rest = bus.split(":", 1) if bus.count(":") == 2 else ("0000", bus)
        path = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}/local_cpulist"
        cpus = set()
        for part in open(path).read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def fwd_flops(l, T=None):
    T = T or l.T
    return 2 * T * l.m * l.n + 2 * T * l.r * (l.n + l.m)


def bwd_flops(l, T=None):
    T = T or l.T
    return 2 * T * l.m * l.n + 4 * T * l.r * (l.n + l.m)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons with NVML during the
    timed region (what nvidia-smi --query-gpu=clocks.sm,... reports)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index, period_s=0.005):
        self.period = period_s
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            uuid = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(device_index).uuid)
            except Exception:
                pass
            self.h = None
            if uuid:
                try:
                    self.h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
                except Exception:
                    self.h = None
            if self.h is None:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[device_index]) if vis and vis.split(",")[0].isdigit() else device_index
                self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"], "samples": 0}
        reasons = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------- oracle leg
def cpu_oracle_sample(wl, target_s=12.0, max_tokens=None):
    """The fp64 oracle, as it stands, on the first R tokens of every linear of
    the workload (a complete R-token fwd+bwd problem).  R is calibrated so the
    sample takes about target_s seconds.  Returns (flops/s, seconds, R, threads)."""
    import oracle
    oracle.build()
    threads = oracle.num_threads()
    inputs = [make_lora_inputs(l.T, l.n, l.m, l.r, seed=2403 + i) for i, l in enumerate(wl.linears)]

    def run(R):
        t0 = time.perf_counter()
        for l, d in zip(wl.linears, inputs):
            x, dy = d["x"][:R], d["dy"][:R]
            oracle.lora_fwd(x, d["w0"], d["a"], d["b"], l.alpha)
            oracle.lora_bwd(x, d["w0"], d["a"], d["b"], dy, l.alpha)
        return time.perf_counter() - t0

    T = wl.linears[0].T
    R = 2
    run(R)  # first touch of the inputs, thread pool start-up
    dt = run(R)
    while dt < 0.5 and R < T:
        R = min(T, R * 4)
        dt = run(R)
    R_target = int(max(1, min(T, max_tokens or T, R * target_s / max(dt, 1e-6))))
    dt = run(R_target)
    return workload_flops(wl, R_target) / dt, dt, R_target, threads


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    K, W = args.steps, args.warmup
    # each step a bounded sample sized so the whole run ends within ~3 minutes
    per_step = max(0.5, min(4.0, 150.0 / max(1, K + W)))
    _, _, R, threads = cpu_oracle_sample(wl, target_s=per_step)
    import oracle
    inputs = [make_lora_inputs(l.T, l.n, l.m, l.r, seed=2403 + i) for i, l in enumerate(wl.linears)]

    def step():
        for l, d in zip(wl.linears, inputs):
            oracle.lora_fwd(d["x"][:R], d["w0"], d["a"], d["b"], l.alpha)
            oracle.lora_bwd(d["x"][:R], d["w0"], d["a"], d["b"], d["dy"][:R], l.alpha)

    for _ in range(W):
        step()
    t0 = time.perf_counter()
    for _ in range(K):
        step()
    dt = time.perf_counter() - t0
    flops = workload_flops(wl, R) * K
    value = flops / dt / 1e12
    sample = (f"first {R} of {wl.linears[0].T} tokens of every linear of {wl.key} "
              f"(complete {R}-token fwd+bwd problems), fp64 C oracle, OpenMP {threads} threads")
    line = {
        "impl": "reference", "metric": "LoRA-linear fwd+bwd TFLOP/s (% bf16 peak) and tokens/s",
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": K, "warmup": W,
        "ms_per_step": dt / K * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.key, "description": wl.description, "sample_tokens": R},
        "tokens_per_s": R * K / dt,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- GPU leg
def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import __graft_entry__
    if local_rank == 0:   # one builder per node (no-op when liblora.so is current)
        __graft_entry__._build_module().build()   # (by path: the package __init__ loads the library)
    if world > 1:
        dist.barrier(device_ids=[local_rank])
    import paper_2403_11366_b200 as L
    from paper_2403_11366_b200 import tp
    L.lora_device_check()

    stream = torch.cuda.current_stream()
    comm = tp.LoraComm() if (world > 1 or args.force_tp) else None

    # ---- inputs (seeded, synthetic, sharded per rank), resident in HBM
    lin = []
    for i, l in enumerate(wl.linears):
        d = make_lora_inputs(l.T, l.n, l.m, l.r, seed=2403 + i)
        mode = tp.MODES[wl.tp_modes[i]]
        spec = tp.ShardSpec(mode, world, rank, l.n, l.m)
        w0, a, b, _ = tp.shard_params(spec, d["w0"], d["a"], d["b"])
        x = tp.shard_input(spec, d["x"])
        dy = tp.shard_output_grad(spec, d["dy"])

        def to_dev(arr):
            arr = np.ascontiguousarray(arr, dtype=np.uint16)
            return torch.from_numpy(arr.view(np.int16)).view(torch.bfloat16).to(dev)

        T, n, m, r = l.T, spec.local_n, spec.local_m, l.r
        e = dict(l=l, spec=spec, x=to_dev(x), w0=to_dev(w0), a=to_dev(a), b=to_dev(b), dy=to_dev(dy),
                 y=torch.empty((T, m), dtype=torch.bfloat16, device=dev),
                 h=torch.empty((T, r), dtype=torch.float32, device=dev),
                 dx=torch.empty((T, n), dtype=torch.bfloat16, device=dev),
                 da=torch.zeros((r, n), dtype=torch.float32, device=dev),
                 db=torch.zeros((m, r), dtype=torch.float32, device=dev))
        dd = L.dims(T, n, m, r, l.alpha)
        import ctypes
        wf = L.lora_linear_fwd_workspace_bytes(dd)
        wb = int(L.lib.lora_tp_linear_bwd_workspace_bytes(ctypes.byref(dd)))
        if args.dropout > 0.0:
            wf = max(wf, int(L.lib.lora_linear_fwd_dropout_workspace_bytes(ctypes.byref(dd))))
            wb = max(wb, int(L.lib.lora_linear_bwd_dropout_workspace_bytes(ctypes.byref(dd))))
        e["ws_f"] = torch.empty(max(256, wf), dtype=torch.uint8, device=dev)
        e["ws_b"] = torch.empty(max(256, wb), dtype=torch.uint8, device=dev)
        lin.append(e)
    # the linears of a group read the SAME activation in the model (q/k/v read the
    # attention input, gate/up the MLP input): one shared x tensor per group
    for gidx in wl.groups:
        for i in gidx[1:]:
            lin[i]["x"] = lin[gidx[0]]["x"]
    launches = {"n": 0}

    # N = 1: the linears that share an input in the model (q,k,v / gate,up) run as
    # one grouped call (one persistent launch per fused GEMM)
    use_groups = comm is None and not args.no_group and args.dropout == 0.0
    if args.dropout > 0.0 and comm is not None:
        raise SystemExit("--dropout is single-GPU only (the TP entry points have no dropout variant)")
    for i, e in enumerate(lin):   # one Philox stream per linear (offset = its index)
        e["drop"] = (args.dropout, 2403, i) if args.dropout > 0.0 else None
    groups = []
    if use_groups:
        for gidx in wl.groups:
            members = [lin[i] for i in gidx]
            ds = (L.lora_dims * len(members))(*[L.dims(e["l"].T, e["spec"].local_n, e["spec"].local_m, e["l"].r,
                                                       e["l"].alpha) for e in members])
            wsf = torch.empty(max(256, int(L.lib.lora_linear_fwd_grouped_workspace_bytes(len(members), ds))),
                              dtype=torch.uint8, device=dev)
            wsb = torch.empty(max(256, int(L.lib.lora_linear_bwd_grouped_workspace_bytes(len(members), ds))),
                              dtype=torch.uint8, device=dev)
            groups.append((members, wsf, wsb))

    def step_grouped(ev=None):
        cur = torch.cuda.current_stream()
        for gi, (members, wsf, _) in enumerate(groups):
            if ev is not None and gi == 0:
                ev["f0"].record(stream)
            L.lora_linear_fwd_grouped([(e["x"], e["w0"], e["a"], e["b"], None) for e in members],
                                      [e["l"].alpha for e in members], outs=[(e["y"], e["h"]) for e in members],
                                      workspace=wsf, stream=cur)
            launches["n"] += L.lora_last_launch_count()
            if ev is not None and gi == 0:
                ev["f1"].record(stream)
        for members, _, wsb in groups:
            L.lora_linear_bwd_grouped([(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["h"]) for e in members],
                                      [e["l"].alpha for e in members],
                                      outs=[(e["dx"], e["da"], e["db"]) for e in members], workspace=wsb,
                                      stream=cur)
            launches["n"] += L.lora_last_launch_count()

    # Tensor parallel (N > 1, or --force-tp): the COLUMN-parallel linears that share an
    # input (q/k/v, gate/up) run as one grouped local forward (no collective in column
    # mode) and one lora_tp_linear_bwd_column_group (their dX partials summed, ONE
    # all-reduce); row-parallel linears (o, down) run one by one.
    tp_groups = []
    if comm is not None and not args.no_group and args.dropout == 0.0:
        for gidx in (wl.groups or tuple((i,) for i in range(len(lin)))):
            members = [lin[i] for i in gidx]
            if len(members) > 1 and all(e["spec"].mode == tp.COLUMN for e in members):
                ds = (L.lora_dims * len(members))(*[L.dims(e["l"].T, e["spec"].local_n, e["spec"].local_m,
                                                           e["l"].r, e["l"].alpha) for e in members])
                wsf = torch.empty(max(256, int(L.lib.lora_linear_fwd_grouped_workspace_bytes(len(members), ds))),
                                  dtype=torch.uint8, device=dev)
                wsb = torch.empty(max(256, int(L.lib.lora_tp_linear_bwd_column_group_workspace_bytes(
                    len(members), ds))), dtype=torch.uint8, device=dev)
                dx_sum = torch.empty_like(members[0]["dx"])
                tp_groups.append((members, wsf, wsb, dx_sum))
            else:
                tp_groups.append((members, None, None, None))

    def step_tp(ev=None):
        cur = torch.cuda.current_stream()
        for gi, (members, wsf, _, _) in enumerate(tp_groups):
            if ev is not None and gi == 0:
                ev["f0"].record(stream)
            if wsf is not None:
                L.lora_linear_fwd_grouped([(e["x"], e["w0"], e["a"], e["b"], None) for e in members],
                                          [e["l"].alpha for e in members],
                                          outs=[(e["y"], e["h"]) for e in members], workspace=wsf, stream=cur)
                launches["n"] += L.lora_last_launch_count()
            else:
                for e in members:
                    tp.tp_linear_fwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["l"].alpha, y=e["y"],
                                     h_out=e["h"], workspace=e["ws_f"], stream=cur)
                    launches["n"] += L.lora_last_launch_count()
            if ev is not None and gi == 0:
                ev["f1"].record(stream)
        for members, _, wsb, dx_sum in tp_groups:
            if wsb is not None:
                tp.tp_linear_bwd_column_group(comm, [e["spec"] for e in members],
                                              [(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["h"]) for e in members],
                                              [e["l"].alpha for e in members], dx_sum=dx_sum,
                                              outs=[(e["dx"], e["da"], e["db"]) for e in members], workspace=wsb,
                                              stream=cur)
                launches["n"] += L.lora_last_launch_count()
            else:
                for e in members:
                    tp.tp_linear_bwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["dy"], e["l"].alpha,
                                     h_saved=e["h"], dx=e["dx"], da=e["da"], db=e["db"], workspace=e["ws_b"],
                                     reduce_lora_grads=True, stream=cur)
                    launches["n"] += L.lora_last_launch_count()

    def step(ev=None):
        if use_groups:
            return step_grouped(ev)
        if tp_groups:
            return step_tp(ev)
        for e in lin:
            if ev is not None and e is lin[0]:
                ev["f0"].record(stream)
            if comm is None:
                L.lora_linear_fwd(e["x"], e["w0"], e["a"], e["b"], e["l"].alpha, y=e["y"], h_out=e["h"],
                                  workspace=e["ws_f"], stream=torch.cuda.current_stream(), dropout=e["drop"])
            else:
                tp.tp_linear_fwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["l"].alpha, y=e["y"],
                                 h_out=e["h"], workspace=e["ws_f"], stream=torch.cuda.current_stream())
            launches["n"] += L.lora_last_launch_count()
            if ev is not None and e is lin[0]:
                ev["f1"].record(stream)
        for e in lin:
            if comm is None:
                L.lora_linear_bwd(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["l"].alpha, h_saved=e["h"],
                                  dx=e["dx"], da=e["da"], db=e["db"], workspace=e["ws_b"],
                                  stream=torch.cuda.current_stream(), dropout=e["drop"])
            else:
                tp.tp_linear_bwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["dy"], e["l"].alpha,
                                 h_saved=e["h"], dx=e["dx"], da=e["da"], db=e["db"], workspace=e["ws_b"],
                                 reduce_lora_grads=True, stream=torch.cuda.current_stream())
            launches["n"] += L.lora_last_launch_count()

    # L2 flush between timed steps, outside the event pairs: write a 2 x L2
    # buffer, then read a second 2 x L2 buffer, so the step starts with a cold
    # L2 that holds no dirty lines (otherwise the first kernel of the step pays
    # for writing the flush data back to HBM)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_w = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_r = torch.zeros_like(flush_w)

    class _Flush:
        def fill_(self, v):
            flush_w.fill_(float(v))
            torch.sum(flush_r)

    flush = _Flush()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        step()
    barrier()

    K = args.steps
    use_graph = args.graph in ("on", "auto")
    graph = None
    if use_graph:
        # the whole step (every fwd + bwd launch, and under TP every NCCL collective)
        # as one CUDA graph, replayed per step -- no host launch cost in the timed loop
        gstream = torch.cuda.Stream(device=dev)
        gstream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        launches["n"] = 0
        try:
            with torch.cuda.stream(gstream):
                with torch.cuda.graph(graph, stream=gstream):
                    step()
        except Exception as ex:   # (symmetric on every rank) -> time the eager step instead
            if args.graph == "on":
                raise
            print(f"bench: CUDA graph capture failed ({ex!r}); timing eager steps", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
        stream.wait_stream(gstream)
        per_step_launches = launches["n"]
    if graph is not None:
        for _ in range(3):
            graph.replay()
        barrier()
        # the graph must really contain the step: clear an output, replay, check it came back
        lin[0]["y"].zero_()
        graph.replay()
        barrier()
        if per_step_launches == 0 or int(torch.count_nonzero(lin[0]["y"]).item()) == 0:
            raise RuntimeError("CUDA graph capture of the step is empty")
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    fev = [dict(f0=torch.cuda.Event(enable_timing=True), f1=torch.cuda.Event(enable_timing=True))
           for _ in range(K)]
    launches["n"] = 0
    with ClockSampler(local_rank) as clk:
        barrier()
        for i in range(K):
            flush.fill_(i & 0xFF)
            ev0[i].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step(None if (use_groups or tp_groups) else fev[i])
            ev1[i].record(stream)
        barrier()
    step_ms = [ev0[i].elapsed_time(ev1[i]) for i in range(K)]
    # roofline kernel: the step's first forward launch -- the grouped fused K1 of the
    # first group of linears (or the first linear's K1 when ungrouped) -- timed with
    # CUDA events on its launching stream inside K further eager steps (same flush)
    if graph is not None:
        launches["n"] = per_step_launches * K
    if graph is not None or use_groups or tp_groups:
        n_before = launches["n"]
        for i in range(K):
            flush.fill_(i & 0xFF)
            step(fev[i])
        launches["n"] = n_before
        barrier()
    fwd_ms = [fev[i]["f0"].elapsed_time(fev[i]["f1"]) for i in range(K)]
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    gpu_launches = launches["n"]

    # ---- end to end through the public API with host buffers
    xs = list({id(e["x"]): e["x"] for e in lin}.values())     # each distinct input once
    # pinned host buffers on the GPU's own NUMA node (first touch by a thread bound to
    # the GPU-local CPUs): a remote node halves the H2D bandwidth on a 2-socket host
    old_aff = os.sched_getaffinity(0)
    local = gpu_local_cpus(local_rank)
    if local:
        os.sched_setaffinity(0, local)
    try:
        hx = [t.cpu().pin_memory() for t in xs]
        hdy = [e["dy"].cpu().pin_memory() for e in lin]
        hda = [torch.zeros_like(e["da"], device="cpu").pin_memory() for e in lin]
        hdb = [torch.zeros_like(e["db"], device="cpu").pin_memory() for e in lin]
    finally:
        if local:
            os.sched_setaffinity(0, old_aff)
    h2d = sum(t.numel() * t.element_size() for t in hx + hdy)
    d2h = sum(t.numel() * t.element_size() for t in hda + hdb)

    # Double-buffered: step i computes from buffer set i % 2 while a copy stream
    # uploads step i+1's inputs into the other set (the H2D copies of every step
    # stay inside the timed region; they overlap the previous step's kernels).
    x_of = [next(j for j, t in enumerate(xs) if t is e["x"]) for e in lin]
    xbuf = [[t, torch.empty_like(t)] for t in xs]
    dybuf = [[e["dy"], torch.empty_like(e["dy"])] for e in lin]
    cstream = torch.cuda.Stream(device=dev)

    def e2e_run(n_steps):
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]
        start = torch.cuda.Event()
        start.record(stream)
        cstream.wait_event(start)

        def upload(k):
            with torch.cuda.stream(cstream):
                for j, a_ in enumerate(hx):
                    xbuf[j][k].copy_(a_, non_blocking=True)
                for i, b_ in enumerate(hdy):
                    dybuf[i][k].copy_(b_, non_blocking=True)
                copied[k].record(cstream)

        upload(0)
        for it in range(n_steps):
            k = it % 2
            stream.wait_event(copied[k])
            for i, e in enumerate(lin):
                e["x"] = xbuf[x_of[i]][k]
                e["dy"] = dybuf[i][k]
            step()
            used[k].record(stream)
            for e, a_, b_ in zip(lin, hda, hdb):
                a_.copy_(e["da"], non_blocking=True)
                b_.copy_(e["db"], non_blocking=True)
            if it + 1 < n_steps:
                if it >= 1:
                    cstream.wait_event(used[1 - k])   # step it-1 is done with that set
                upload(1 - k)

    e2e_run(3)
    barrier()
    Ke = max(3, min(K, 50))
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    e2e_run(Ke)
    s1.record(stream)
    barrier()
    for i, e in enumerate(lin):   # back to the original buffers
        e["x"] = xbuf[x_of[i]][0]
        e["dy"] = dybuf[i][0]
    e2e_ms = s0.elapsed_time(s1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- the HBM-bound kernels of the path, timed alone (report them in
    # GB/s against the measured HBM bandwidth): K4 merge of the first linear, and the
    # gradient-only backward (B^T pack + h split, gh row projection + split, K3) -- L2 flushed before each call
    aux = {}
    if world == 1:
        e = lin[0]
        l0_ = e["l"]
        w_out = torch.empty_like(e["w0"])
        da_, db_ = torch.empty_like(e["da"]), torch.empty_like(e["db"])

        def timed(fn, reps=20):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(reps):
                flush.fill_(1)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                fn()
                a1.record(stream)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(a1) * 1e-3)
            return float(np.median(ts))

        T0, n0, m0, r0 = l0_.T, l0_.n, l0_.m, l0_.r
        t_merge = timed(lambda: L.lora_merge(e["w0"], e["a"], e["b"], l0_.alpha, w_out=w_out,
                                             stream=torch.cuda.current_stream()))
        t_grads = timed(lambda: L.lora_linear_bwd(e["x"], e["w0"], e["a"], e["b"], e["dy"], l0_.alpha,
                                                  h_saved=e["h"], want_dx=False, da=da_, db=db_,
                                                  workspace=e["ws_b"], stream=torch.cuda.current_stream()))
        # N3: one Adam step over every adapter tensor of the workload (A and B of each
        # linear, fp32 master + moments): ONE launch; 30 bytes per parameter
        ad = []
        for e in lin:
            for t, g in ((e["a"], e["da"]), (e["b"], e["db"])):
                ad.append((t.clone(), g, torch.zeros_like(g), torch.zeros_like(g), t.float()))
        adam_step_no = [0]

        def adam_call():
            adam_step_no[0] += 1
            L.lora_adam_step(ad, adam_step_no[0], 1e-4, stream=torch.cuda.current_stream())

        t_adam = timed(adam_call)
        adam_bytes = 30 * sum(t[0].numel() for t in ad)
        merge_bytes = 4 * m0 * n0 + 2 * r0 * (m0 + n0)
        # dY read twice (gh pre-pass, dB), x once, coefficients ~ 16 T r
        grads_bytes = 2 * T0 * (2 * m0 + n0) + 16 * T0 * r0
        aux = {"merge": {"us": t_merge * 1e6, "bytes": merge_bytes, "gbs": merge_bytes / t_merge / 1e9},
               "adam_all_adapters": {"us": t_adam * 1e6, "bytes": adam_bytes, "gbs": adam_bytes / t_adam / 1e9,
                                     "tensors": len(ad)},
               "grads_only": {"us": t_grads * 1e6, "bytes": grads_bytes, "gbs": grads_bytes / t_grads / 1e9,
                              "kernels": "B^T pack + h split, gh row projection + gh split, K3 (lora_linear_bwd, dx = NULL)"}}

    # ---- report (rank 0)
    if rank == 0:
        peaks, peak_src = load_peaks()
        flops_step = workload_flops(wl)
        value = flops_step * K / (total_ms * 1e-3) / 1e12
        tokens = wl.linears[0].T
        l0 = wl.linears[0]
        roof_linears = ([lin[i]["l"] for i in wl.groups[0]] if (use_groups or tp_groups) and wl.groups else [l0])
        f_fwd = sum(fwd_flops(l) for l in roof_linears) / world
        fwd_avg_s = float(np.mean(fwd_ms)) * 1e-3
        achieved = f_fwd / fwd_avg_s / 1e12
        peak = peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
        traffic = None
        tp_path = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp_path):
            tj = json.load(open(tp_path))
            traffic = (tj.get("grouped_fwd_bytes_per_launch", {}).get(wl.key) if use_groups
                       else tj.get("fused_fwd_bytes_per_launch_single"))
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cval, cdt, R, thr = cpu_oracle_sample(wl, target_s=args.cpu_seconds)
            cpu = {"value": cval / 1e12, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
                   "sample": f"first {R} of {tokens} tokens of every linear of {wl.key} (complete "
                             f"{R}-token fwd+bwd problems), fp64 C oracle, {cdt:.1f} s"}
        line = {
            "metric": "LoRA-linear fwd+bwd TFLOP/s (% bf16 peak) and tokens/s",
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl.key, "description": wl.description,
                       "linears": [f"{l.name}:{l.n}->{l.m}" for l in wl.linears],
                       "tokens": tokens, "rank": l0.r, "alpha": l0.alpha,
                       "global_batch": 1, "seq_len": tokens,
                       "parallelism": f"tp{world}" if comm is not None else "single",
                       "cuda_graph": graph is not None,
                       "grouped_calls": ([[wl.linears[i].name for i in g] for g in wl.groups]
                                         if (use_groups or tp_groups) else None),
                       "shared_inputs": [[wl.linears[i].name for i in g] for g in wl.groups if len(g) > 1],
                       "lora_dropout": args.dropout,
                       "l2": "flushed between timed steps (2xL2 write then 2xL2 read, outside the "
                             "event pairs)"},
            "tokens_per_s": tokens * K / (total_ms * 1e-3),
            "pct_of_bf16_peak": value / (peak * world) * 100.0,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": (f"lora_linear_fwd_grouped of {[l.name for l in roof_linears]} (one fused K1 "
                                    f"launch) inside the step, " if len(roof_linears) > 1 else
                                    f"lora_linear_fwd of '{l0.name}' (B6 pack + fused K1) inside the step, ") +
                                   f"{f_fwd / 1e9:.2f} algorithmic GFLOP per launch, avg {fwd_avg_s * 1e6:.1f} us",
                         "peak_source": peak_src + " bf16_tflops (burst)"},
            "step_ms_median": float(np.median(step_ms)),
            "cpu_baseline": cpu,
            "e2e": {"value": flops_step * Ke / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
        if aux:
            hbm = peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
            for v in aux.values():
                v["frac_of_hbm"] = v["gbs"] / hbm
            line["hbm_bound_kernels"] = dict(aux, hbm_peak_gbs=hbm, linear=l0.name)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-tp", action="store_true",
                    help="run the tensor-parallel code path (NCCL communicator, TP entry points) even at N = 1")
    ap.add_argument("--dropout", type=float, default=0.0,
                    help="LoRA dropout p (Listing 3 LORA_DROPOUT = 0.05); 0 = the north-star path")
    ap.add_argument("--no-group", action="store_true",
                    help="one call per linear instead of grouped calls for linears sharing an input")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each step as one CUDA graph (auto: at N = 1)")
    args = ap.parse_args()
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, wl)
    return run_ours(args, wl)


if __name__ == "__main__":
    sys.exit(main())

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
parallel q/k/v/gate/up, row parallel o/down) over N processes launched by
torchrun: strong scaling, NCCL all-reduces inside the step.  The default
workload is cfg2 at N = 1 and cfg3 (the 7B decoder-layer LoRA set BASELINE.json
names for 2/4/8 GPUs) at N > 1.

Prints ONE JSON line on rank 0.  `--impl reference` times the fp64 CPU oracle
(oracle/, the parity reference) on a bounded token sample of the same workload.
The timed step (StepRunner) is importable: tests/test_gpu_bench_path.py checks
exactly this step -- the same calls, buffers and CUDA graph -- against the oracle.
"""
from __future__ import annotations

import argparse
import ctypes
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
METRIC = "LoRA-linear fwd+bwd TFLOP/s (% bf16 peak) and tokens/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def workload_flops(wl, T=None):
    return sum(algorithmic_flops(T or l.T, l.n, l.m, l.r) for l in wl.linears)


def fwd_flops(l, T=None):
    T = T or l.T
    return 2 * T * l.m * l.n + 2 * T * l.r * (l.n + l.m)


def bwd_dx_flops(l, T=None):
    """The fused dX kernel (K2): dY W0 + gh A and gh = s dY B."""
    T = T or l.T
    return 2 * T * l.m * l.n + 2 * T * l.r * (l.n + l.m)


def cpu_model_name():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


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


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons with NVML during the
    timed region (what nvidia-smi --query-gpu=clocks.sm,... reports)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index, period_s=0.002):
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
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": K, "warmup": W,
        "ms_per_step": dt / K * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.key, "description": wl.description, "sample_tokens": R},
        "tokens_per_s": R * K / dt,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu_model": cpu_model_name()},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- the timed step
def _bits_to_dev(bits, dev):
    import torch
    arr = np.ascontiguousarray(bits, dtype=np.uint16)
    return torch.from_numpy(arr.view(np.int16)).view(torch.bfloat16).to(dev)


class StepRunner:
    """One step of the workload: forward + backward of every LoRA linear, through
    the public C ABI (via the binding), exactly as bench.py times it.

    N = 1: the linears that read the same input in the model (q/k/v, gate/up)
    share ONE x tensor and run as one grouped call each for fwd and bwd (one
    persistent launch per fused GEMM).  TP (N > 1 or force_tp): column-parallel
    groups run the grouped local forward + lora_tp_linear_bwd_column_group
    (their dX partials summed, ONE all-reduce); row-parallel linears run
    lora_tp_linear_fwd/bwd (y all-reduce / dB all-reduce).

    `nsets` buffer sets of the step's inputs (x, dY) and outputs (y, dX) exist;
    `use_set(k)` points the step at set k (the e2e leg captures one CUDA graph per
    set and double-buffers host transfers against compute).  The numpy bit
    patterns of the unsharded inputs stay in `host` for the parity checks."""

    def __init__(self, wl, dev, world=1, rank=0, comm=None, group=True, dropout=0.0, nsets=1, seed0=2403,
                 comm_mode="nccl", keep_mask="kept"):
        import torch

        import paper_2403_11366_b200 as L
        from paper_2403_11366_b200 import tp
        self.L, self.tp, self.torch = L, tp, torch
        self.wl, self.dev, self.world, self.rank, self.comm = wl, dev, world, rank, comm
        self.launches = 0
        self.host = []
        lin = []
        for i, l in enumerate(wl.linears):
            d = make_lora_inputs(l.T, l.n, l.m, l.r, seed=seed0 + i)
            self.host.append(d)
        # the linears of a group read the SAME activation in the model
        for gidx in wl.groups:
            for i in gidx[1:]:
                self.host[i]["x"] = self.host[gidx[0]]["x"]
        for i, l in enumerate(wl.linears):
            d = self.host[i]
            mode = tp.MODES[wl.tp_modes[i]]
            spec = tp.ShardSpec(mode, world, rank, l.n, l.m)
            w0, a, b, _ = tp.shard_params(spec, d["w0"], d["a"], d["b"])
            T, n, m, r = l.T, spec.local_n, spec.local_m, l.r
            e = dict(l=l, spec=spec, w0=_bits_to_dev(w0, dev), a=_bits_to_dev(a, dev), b=_bits_to_dev(b, dev),
                     h=torch.empty((T, r), dtype=torch.float32, device=dev))
            e["da_sets"] = [torch.zeros((r, n), dtype=torch.float32, device=dev) for _ in range(nsets)]
            e["db_sets"] = [torch.zeros((m, r), dtype=torch.float32, device=dev) for _ in range(nsets)]
            e["dy_sets"] = [_bits_to_dev(tp.shard_output_grad(spec, d["dy"]), dev)]
            e["y_sets"] = [torch.empty((T, m), dtype=torch.bfloat16, device=dev) for _ in range(nsets)]
            e["dx_sets"] = [torch.empty((T, n), dtype=torch.bfloat16, device=dev) for _ in range(nsets)]
            dd = L.dims(T, n, m, r, l.alpha)
            wf = L.lora_linear_fwd_workspace_bytes(dd)
            wb = int(L.lib.lora_tp_linear_bwd_workspace_bytes(ctypes.byref(dd)))
            if dropout > 0.0:
                wf = max(wf, int(L.lib.lora_linear_fwd_dropout_workspace_bytes(ctypes.byref(dd))))
                wb = max(wb, int(L.lib.lora_linear_bwd_dropout_workspace_bytes(ctypes.byref(dd))),
                         int(L.lib.lora_tp_linear_bwd_dropout_workspace_bytes(ctypes.byref(dd))))
            e["ws_f"] = torch.empty(max(256, wf), dtype=torch.uint8, device=dev)
            e["ws_b"] = torch.empty(max(256, wb), dtype=torch.uint8, device=dev)
            # one Philox stream per linear; keep_mask "kept": the forward stores the keep bits
            # (T n / 8 bytes, lora_dropout.keep_bits) and M . x (lora_dropout.masked_x), the
            # backward reads them instead of drawing and masking again
            e["drop"] = None
            if dropout > 0.0:
                e["drop"] = (dropout, 2403, i) + ((L.dropout_keep_bits(T, n, dev),
                                                   torch.empty((T, n), dtype=torch.bfloat16, device=dev))
                                                  if keep_mask == "kept" else ())
            lin.append(e)
        for gidx in wl.groups:   # one shared x tensor per group (per set)
            x0 = _bits_to_dev(tp.shard_input(lin[gidx[0]]["spec"], self.host[gidx[0]]["x"]), dev)
            for i in gidx:
                lin[i]["x_sets"] = [x0]
        for _ in range(1, nsets):
            for gidx in wl.groups:
                xk = torch.empty_like(lin[gidx[0]]["x_sets"][0])
                for i in gidx:
                    lin[i]["x_sets"].append(xk)
            for e in lin:
                e["dy_sets"].append(torch.empty_like(e["dy_sets"][0]))
        # TP: the LoRA gradients that are partial sums on each rank (column: dA, row: dB;
        # DESIGN.md R11-R12) are views of ONE flat fp32 bucket per buffer set, reduced by a
        # single all-reduce at the end of the step instead of one per linear
        self.grad_bucket = None
        if comm is not None:
            sizes = [(e["l"].r * e["spec"].local_n) if e["spec"].mode == tp.COLUMN
                     else (e["spec"].local_m * e["l"].r) for e in lin]
            total = sum(sizes)
            self.grad_bucket = [torch.zeros(total, dtype=torch.float32, device=dev) for _ in range(nsets)]
            for k in range(nsets):
                off = 0
                for e, sz in zip(lin, sizes):
                    view = self.grad_bucket[k][off:off + sz]
                    if e["spec"].mode == tp.COLUMN:
                        e["da_sets"][k] = view.view(e["l"].r, e["spec"].local_n)
                    else:
                        e["db_sets"][k] = view.view(e["spec"].local_m, e["l"].r)
                    off += sz
        self.lin = lin
        self.nsets = nsets
        self.use_set(0)

        self.use_groups = comm is None and group
        self.dropout = dropout
        # (--dropout under TP: grouped column members through lora_linear_fwd_grouped_dropout and
        # lora_tp_linear_bwd_column_group_dropout, row linears through lora_tp_linear_{fwd,bwd}_dropout)
        self.groups = []
        if self.use_groups:
            for gidx in wl.groups:
                members = [lin[i] for i in gidx]
                ds = self._dims(members)
                if dropout > 0.0:
                    nf = int(L.lib.lora_linear_fwd_grouped_dropout_workspace_bytes(len(members), ds))
                    nb = int(L.lib.lora_linear_bwd_grouped_dropout_workspace_bytes(len(members), ds))
                else:
                    nf = int(L.lib.lora_linear_fwd_grouped_workspace_bytes(len(members), ds))
                    nb = int(L.lib.lora_linear_bwd_grouped_workspace_bytes(len(members), ds))
                wsf = torch.empty(max(256, nf), dtype=torch.uint8, device=dev)
                wsb = torch.empty(max(256, nb), dtype=torch.uint8, device=dev)
                self.groups.append((members, wsf, wsb))
        self.tp_groups = []
        if comm is not None and group:
            for gidx in (wl.groups or tuple((i,) for i in range(len(lin)))):
                members = [lin[i] for i in gidx]
                if len(members) > 1 and all(e["spec"].mode == tp.COLUMN for e in members):
                    ds = self._dims(members)
                    if dropout > 0.0:
                        nf = L.lib.lora_linear_fwd_grouped_dropout_workspace_bytes(len(members), ds)
                        nb = L.lib.lora_tp_linear_bwd_column_group_dropout_workspace_bytes(len(members), ds)
                    else:
                        nf = L.lib.lora_linear_fwd_grouped_workspace_bytes(len(members), ds)
                        nb = L.lib.lora_tp_linear_bwd_column_group_workspace_bytes(len(members), ds)
                    wsf = torch.empty(max(256, int(nf)), dtype=torch.uint8, device=dev)
                    wsb = torch.empty(max(256, int(nb)), dtype=torch.uint8, device=dev)
                    dx_sum = [torch.empty_like(members[0]["dx_sets"][0]) for _ in range(nsets)]
                    self.tp_groups.append((members, wsf, wsb, dx_sum))
                else:
                    self.tp_groups.append((members, None, None, None))
        # comm-fused epilogues (lora_symm): one symmetric buffer per
        # rank holding, per row-parallel linear, its partial y and the reduced y, and per
        # column group its members' dX partials and the reduced dX w.r.t. the input
        self.symm = None
        self.comm_mode = comm_mode if comm is not None else "none"
        if self.comm_mode == "fused":
            if dropout > 0.0:
                raise SystemExit("--comm fused has no LoRA-dropout variant (use --comm nccl)")
            if not self.tp_groups:
                raise SystemExit("--comm fused needs the grouped TP step (no --no-group / --dropout)")
            off, regions = 0, []

            def region(nbytes):
                nonlocal off
                o = off
                off += (nbytes + 255) // 256 * 256
                return o

            for members, wsf, wsb, dx_sum in self.tp_groups:
                if wsb is not None:
                    T, n = members[0]["l"].T, members[0]["spec"].local_n
                    regions.append(("col", members, region(len(members) * T * n * 2), region(T * n * 2)))
                else:
                    for e in members:
                        if e["spec"].mode == tp.ROW:
                            T, m = e["l"].T, e["spec"].local_m
                            regions.append(("row", e, region(T * m * 2), region(T * m * 2)))
            self.symm = tp.SymmBuffer(off + 4096)
            self.fused_regions = {}
            for kind, obj, part, out in regions:
                if kind == "row":
                    self.fused_regions[id(obj)] = (part, out)
                    T, m = obj["l"].T, obj["spec"].local_m
                    obj["y_sets"] = [self.symm.view(out, (T, m))] * nsets   # y lives in the symmetric buffer
                else:
                    self.fused_regions[id(obj[0])] = (part, out)
            self.use_set(self.k)

    def _dims(self, members):
        L = self.L
        return (L.lora_dims * len(members))(*[L.dims(e["l"].T, e["spec"].local_n, e["spec"].local_m, e["l"].r,
                                                     e["l"].alpha) for e in members])

    def use_set(self, k):
        self.k = k
        for e in self.lin:
            e["x"], e["dy"], e["y"], e["dx"] = e["x_sets"][k], e["dy_sets"][k], e["y_sets"][k], e["dx_sets"][k]
            e["da"], e["db"] = e["da_sets"][k], e["db_sets"][k]

    def distinct_x(self, k=0):
        return list({id(e["x_sets"][k]): e["x_sets"][k] for e in self.lin}.values())

    # ------------------------------------------------------------ one step
    def step(self, ev=None):
        """ev (optional): dict of torch.cuda.Events -- f0/f1 around the first forward
        call, k2a/k2b and k3a/k3b around the first backward call's dX and dA/dB
        kernels (lora_profile_next_bwd)."""
        if self.use_groups:
            return self._step_grouped(ev)
        if self.tp_groups:
            return self._step_tp(ev)
        return self._step_single(ev)

    def _prof_bwd(self, ev):
        if ev is not None and "k2a" in ev:
            self.L.lora_profile_next_bwd(ev["k2a"], ev["k2b"], ev["k3a"], ev["k3b"])

    def _step_grouped(self, ev):
        L = self.L
        cur = self.torch.cuda.current_stream()
        for gi, (members, wsf, _) in enumerate(self.groups):
            if ev is not None and gi == 0:
                ev["f0"].record(cur)
            drops = [e["drop"] for e in members] if self.dropout > 0.0 else None
            L.lora_linear_fwd_grouped([(e["x"], e["w0"], e["a"], e["b"], None) for e in members],
                                      [e["l"].alpha for e in members], outs=[(e["y"], e["h"]) for e in members],
                                      workspace=wsf, stream=cur, dropouts=drops)
            self.launches += L.lora_last_launch_count()
            if ev is not None and gi == 0:
                ev["f1"].record(cur)
        for gi, (members, _, wsb) in enumerate(self.groups):
            if gi == 0:
                self._prof_bwd(ev)
            drops = [e["drop"] for e in members] if self.dropout > 0.0 else None
            L.lora_linear_bwd_grouped([(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["h"]) for e in members],
                                      [e["l"].alpha for e in members],
                                      outs=[(e["dx"], e["da"], e["db"]) for e in members], workspace=wsb, stream=cur,
                                      dropouts=drops)
            self.launches += L.lora_last_launch_count()

    def _step_tp(self, ev):
        L, tp, comm = self.L, self.tp, self.comm
        cur = self.torch.cuda.current_stream()
        fused = self.comm_mode == "fused"
        for gi, (members, wsf, _, _) in enumerate(self.tp_groups):
            if ev is not None and gi == 0:
                ev["f0"].record(cur)
            if wsf is not None:
                drops = [e["drop"] for e in members] if self.dropout > 0.0 else None
                L.lora_linear_fwd_grouped([(e["x"], e["w0"], e["a"], e["b"], None) for e in members],
                                          [e["l"].alpha for e in members],
                                          outs=[(e["y"], e["h"]) for e in members], workspace=wsf, stream=cur,
                                          dropouts=drops)
                self.launches += L.lora_last_launch_count()
            else:
                for e in members:
                    if fused and e["spec"].mode == tp.ROW:   # y all-reduce fused into the GEMM
                        part, out = self.fused_regions[id(e)]
                        tp.tp_linear_fwd_fused(self.symm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["l"].alpha,
                                               part_offset=part, y_offset=out, h_out=e["h"], workspace=e["ws_f"],
                                               stream=cur)
                    else:
                        tp.tp_linear_fwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["l"].alpha,
                                         y=e["y"], h_out=e["h"], workspace=e["ws_f"], stream=cur,
                                         dropout=e["drop"])
                    self.launches += L.lora_last_launch_count()
            if ev is not None and gi == 0:
                ev["f1"].record(cur)
        for gi, (members, _, wsb, dx_sum) in enumerate(self.tp_groups):
            if gi == 0:
                self._prof_bwd(ev)
            if wsb is not None and fused:   # dX all-reduce (over ranks and members) fused into K2
                part, out = self.fused_regions[id(members[0])]
                tp.tp_linear_bwd_column_group_fused(self.symm, [e["spec"] for e in members],
                                                    [(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["h"])
                                                     for e in members], [e["l"].alpha for e in members],
                                                    comm=comm, part_offset=part, dx_offset=out,
                                                    outs=[(e["da"], e["db"]) for e in members],
                                                    reduce_lora_grads=False, workspace=wsb, stream=cur)
                self.launches += L.lora_last_launch_count()
            elif wsb is not None:
                tp.tp_linear_bwd_column_group(comm, [e["spec"] for e in members],
                                              [(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["h"]) for e in members],
                                              [e["l"].alpha for e in members], dx_sum=dx_sum[self.k],
                                              outs=[(e["dx"], e["da"], e["db"]) for e in members], workspace=wsb,
                                              reduce_lora_grads=False, stream=cur,
                                              dropouts=[e["drop"] for e in members] if self.dropout > 0.0 else None)
                self.launches += L.lora_last_launch_count()
            else:
                for e in members:
                    tp.tp_linear_bwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["dy"], e["l"].alpha,
                                     h_saved=e["h"], dx=e["dx"], da=e["da"], db=e["db"], workspace=e["ws_b"],
                                     reduce_lora_grads=False, stream=cur, dropout=e["drop"])
                    self.launches += L.lora_last_launch_count()
        comm.allreduce(self.grad_bucket[self.k], stream=cur)   # every partial LoRA gradient of the step

    def _step_single(self, ev):
        L, tp, comm = self.L, self.tp, self.comm
        cur = self.torch.cuda.current_stream()
        lin = self.lin
        for e in lin:
            if ev is not None and e is lin[0]:
                ev["f0"].record(cur)
            if comm is None:
                L.lora_linear_fwd(e["x"], e["w0"], e["a"], e["b"], e["l"].alpha, y=e["y"], h_out=e["h"],
                                  workspace=e["ws_f"], stream=cur, dropout=e["drop"])
            else:
                tp.tp_linear_fwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["l"].alpha, y=e["y"],
                                 h_out=e["h"], workspace=e["ws_f"], stream=cur, dropout=e["drop"])
            self.launches += L.lora_last_launch_count()
            if ev is not None and e is lin[0]:
                ev["f1"].record(cur)
        for e in lin:
            if e is lin[0]:
                self._prof_bwd(ev)
            if comm is None:
                L.lora_linear_bwd(e["x"], e["w0"], e["a"], e["b"], e["dy"], e["l"].alpha, h_saved=e["h"],
                                  dx=e["dx"], da=e["da"], db=e["db"], workspace=e["ws_b"], stream=cur,
                                  dropout=e["drop"])
            else:
                tp.tp_linear_bwd(comm, e["spec"], e["x"], e["w0"], e["a"], e["b"], e["dy"], e["l"].alpha,
                                 h_saved=e["h"], dx=e["dx"], da=e["da"], db=e["db"], workspace=e["ws_b"],
                                 reduce_lora_grads=False, stream=cur, dropout=e["drop"])
            self.launches += L.lora_last_launch_count()
        if comm is not None:
            comm.allreduce(self.grad_bucket[self.k], stream=cur)   # every partial LoRA gradient of the step

    def capture(self, k=0):
        """The whole step (every fwd + bwd launch, and under TP every NCCL
        collective) on buffer set k as one CUDA graph; returns (graph, launches
        per replay)."""
        torch = self.torch
        self.use_set(k)
        cur = torch.cuda.current_stream()
        gstream = torch.cuda.Stream(device=self.dev)
        gstream.wait_stream(cur)
        graph = torch.cuda.CUDAGraph()
        n0 = self.launches
        with torch.cuda.stream(gstream):
            with torch.cuda.graph(graph, stream=gstream):
                self.step()
        cur.wait_stream(gstream)
        return graph, self.launches - n0

    # ------------------------------------------------------------ parity
    def parity(self, rows_per_linear=None, seed=7):
        """The outputs currently in buffer set self.k against the fp64 oracle on the
        same (unsharded) inputs: y, h and dX on sampled token rows (the first 256 --
        one full CTA-pair tile --, 128 random and the last 32), dA and dB in full.
        Only for the unsharded step (N = 1, not TP).  Returns a dict of relF maxima
        over the linears plus the tolerance verdict."""
        import oracle

        from tests.gpu_util import host_f64 as to_f64
        from tests.gpu_util import relF
        if self.world != 1:
            return None
        self.torch.cuda.synchronize()
        worst = {"y": 0.0, "h": 0.0, "dx": 0.0, "da": 0.0, "db": 0.0}
        nrows = 0
        # comm-fused column groups keep only the reduced dX w.r.t. their shared input
        # (the members' partials live in the symmetric buffer): check that sum
        fused_dx = {}
        if self.comm_mode == "fused":
            for members, _, wsb, _ in self.tp_groups:
                if wsb is not None:
                    part, out = self.fused_regions[id(members[0])]
                    T, n = members[0]["l"].T, members[0]["spec"].local_n
                    for e in members:
                        fused_dx[id(e)] = (members, self.symm.view(out, (T, n)))
        dx_sums = {}
        for i, e in enumerate(self.lin):
            l, d = e["l"], self.host[i]
            T = l.T
            if rows_per_linear is None:
                rng = np.random.default_rng(seed + (0 if fused_dx else i))   # (a group's members: same rows)
                rows = np.unique(np.concatenate([np.arange(min(256, T)), rng.choice(T, min(128, T), replace=False),
                                                 np.arange(max(0, T - 32), T)]))
            else:
                rows = rows_per_linear
            kw = {"dropout": e["drop"][:3]} if e["drop"] is not None else {}   # (LoRA dropout: the same mask)
            yo, ho = oracle.lora_fwd(d["x"], d["w0"], d["a"], d["b"], l.alpha, rows=rows, **kw)
            go = oracle.lora_bwd(d["x"], d["w0"], d["a"], d["b"], d["dy"], l.alpha, rows=rows, **kw)
            ri = self.torch.as_tensor(rows, device=self.dev)
            got = {"y": to_f64(e["y"][ri]), "h": to_f64(e["h"][ri]), "da": to_f64(e["da"]), "db": to_f64(e["db"])}
            ref = {"y": yo, "h": ho, "da": go["da"], "db": go["db"]}
            if id(e) in fused_dx:
                members, view = fused_dx[id(e)]
                acc = dx_sums.setdefault(id(members[0]), [None, 0, view])
                acc[0] = go["dx"] if acc[0] is None else acc[0] + go["dx"]
                acc[1] += 1
                if acc[1] == len(members):   # every member's oracle dX rows summed
                    got["dx"], ref["dx"] = to_f64(view[ri]), acc[0]
            else:
                got["dx"], ref["dx"] = to_f64(e["dx"][ri]), go["dx"]
            for k in ref:
                worst[k] = max(worst[k], relF(got[k], ref[k]))
            nrows += len(rows)
        ok = worst["y"] <= 1e-2 and worst["dx"] <= 1e-2 and worst["da"] <= 2e-2 and worst["db"] <= 2e-2
        return {"relF_max_over_linears": worst, "rows_checked_per_linear": int(nrows // len(self.lin)),
                "tolerance": {"y": 1e-2, "dx": 1e-2, "da": 2e-2, "db": 2e-2}, "pass": bool(ok),
                "what": "last timed CUDA-graph replay vs fp64 oracle: y, h, dX on the first 256 + 128 random + "
                        "last 32 token rows of every linear, dA and dB in full"}


# --------------------------------------------------- decoder-layer workload (N4)
LAYERS = {   # the Llama-2 decoder layer at the RAFT sequence length
    "layer7b": dict(T=4096, d=4096, f=11008, heads=32, head_dim=128, r=16, alpha=16.0,
                    description="Llama-2-7B decoder layer, LoRA r=16 on q,k,v,o,gate,up,down, seq 4096"),
    "layer13b": dict(T=4096, d=5120, f=13824, heads=40, head_dim=128, r=8, alpha=16.0,
                     description="Llama-2-13B decoder layer, LoRA r=8 on all seven projections, seq 4096"),
}


def run_layer(args, key):
    """One decoder-layer train step (forward + backward of every piece) per step,
    timed like the linear workloads (CUDA events, L2 flushed outside the events,
    CUDA graph when capture works; max over ranks).  Under torchrun (or with
    --force-tp at N = 1) the layer is tensor-parallel: q/k/v and
    gate/up column-sharded (heads and FFN split), o and down row-sharded."""
    import torch
    import torch.distributed as dist

    from paper_2403_11366_b200 import tp
    from paper_2403_11366_b200.layer import LlamaLayerLoRA, layer_flops
    from synth import make_layer_inputs
    c = LAYERS[key]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import __graft_entry__
    if local_rank == 0:
        __graft_entry__._build_module().build()
    if world > 1:
        dist.barrier(device_ids=[local_rank])
    import paper_2403_11366_b200 as L
    L.lora_device_check()
    bits = make_layer_inputs(c["T"], c["d"], c["f"], c["heads"], c["r"], seed=2403)
    cfg = dict(heads=c["heads"], head_dim=c["head_dim"], eps=1e-5, theta=10000.0, alpha=c["alpha"], ffn=c["f"])
    comm = tp.LoraComm() if (world > 1 or args.force_tp) else None
    if comm is not None:   # this rank's shards (R10-R11)
        d_, f_ = c["d"], c["f"]
        shard = {}
        for p in ("q", "k", "v", "gate", "up", "o", "down"):
            mode = tp.ROW if p in ("o", "down") else tp.COLUMN
            n_, m_ = {"gate": (d_, f_), "up": (d_, f_), "down": (f_, d_)}.get(p, (d_, d_))
            spec = tp.ShardSpec(mode, world, rank, n_, m_)
            shard["w0_" + p], shard["a_" + p], shard["b_" + p], _ = tp.shard_params(
                spec, bits["w0_" + p], bits["a_" + p], bits["b_" + p])
        shard["g1"], shard["g2"] = bits["g1"], bits["g2"]
        params = {k: _bits_to_dev(v, dev) for k, v in shard.items()}
    else:
        params = {k: _bits_to_dev(v, dev) for k, v in bits.items() if k not in ("x", "dout")}
    x, dout = _bits_to_dev(bits["x"], dev), _bits_to_dev(bits["dout"], dev)
    layer = LlamaLayerLoRA(params, cfg, comm=comm)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_w = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_r = torch.zeros_like(flush_w)

    def step():
        layer.forward(x)
        layer.backward(dout)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    graph = None
    if args.graph != "off":
        try:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(graph, stream=s):
                    step()
            torch.cuda.current_stream().wait_stream(s)
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as ex:
            print(f"bench: layer graph capture failed ({ex!r}); timing eager steps", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier(device_ids=[local_rank])
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(K):
            flush_w.fill_(float(i & 0xFF))
            torch.sum(flush_r)
            ev[i][0].record()
            if graph is not None:
                graph.replay()
            else:
                step()
            ev[i][1].record()
        torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    total = float(np.sum(ms))
    if world > 1:
        t = torch.tensor([total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    fl = layer_flops(c["T"], c["d"], c["f"], c["heads"], c["head_dim"], c["r"])
    peaks, peak_src = load_peaks()
    value = fl * K / (total * 1e-3) / 1e12
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    print(json.dumps({
        "metric": "LoRA Llama-2 decoder-layer fwd+bwd TFLOP/s and tokens/s", "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": total / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": key, "description": c["description"], "tokens": c["T"], "rank": c["r"],
                   "parallelism": f"tp{world}" if comm is not None else "single",
                   "cuda_graph": graph is not None, "attention": "cuDNN SDPA (causal), library call",
                   "l2": "flushed between timed steps (outside the event pairs)"},
        "tokens_per_s": c["T"] * K / (total * 1e-3),
        "pct_of_bf16_peak": value / (peaks["bf16_tflops"] * world) * 100.0,
        "flops_per_step": fl, "peak_source": peak_src,
        "step_ms_median": float(np.median(ms)), "clocks": clk.summary()}), flush=True)
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
    R = StepRunner(wl, dev, world, rank, comm, group=not args.no_group, dropout=args.dropout, nsets=2,
                   comm_mode=args.comm, keep_mask=args.dropout_mask)
    lin = R.lin

    # L2 flush between timed steps, outside the event pairs: write a 2 x L2
    # buffer, then read a second 2 x L2 buffer, so the step starts with a cold
    # L2 that holds no dirty lines (otherwise the first kernel of the step pays
    # for writing the flush data back to HBM)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_w = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_r = torch.zeros_like(flush_w)

    def flush(v):
        flush_w.fill_(float(v))
        torch.sum(flush_r)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    R.use_set(0)
    for _ in range(max(3, args.warmup)):
        R.step()
    barrier()

    K = args.steps
    graph = None
    per_step_launches = None
    if args.graph in ("on", "auto"):
        try:
            graph, per_step_launches = R.capture(0)
        except Exception as ex:   # (symmetric on every rank) -> time the eager step instead
            if args.graph == "on":
                raise
            print(f"bench: CUDA graph capture failed ({ex!r}); timing eager steps", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    R.use_set(0)
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
    R.launches = 0
    with ClockSampler(local_rank) as clk:
        barrier()
        for i in range(K):
            flush(i & 0xFF)
            ev0[i].record(stream)
            if graph is not None:
                graph.replay()
            else:
                R.step()
            ev1[i].record(stream)
        barrier()
    step_ms = [ev0[i].elapsed_time(ev1[i]) for i in range(K)]
    gpu_launches = per_step_launches * K if graph is not None else R.launches
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # ---- parity of the timed path itself: the outputs of the last timed replay vs the oracle
    parity = None
    if world == 1 and not args.no_parity:
        parity = R.parity()

    # ---- in-step kernel timing: K further eager steps (same flush), CUDA events on the
    # launching stream around the first group's fused forward (K1) and, through the
    # library's lora_profile_next_bwd hook, around its dX kernel (K2) and dA/dB kernel (K3)
    names = ("f0", "f1", "k2a", "k2b", "k3a", "k3b")
    fev = [{k: torch.cuda.Event(enable_timing=True) for k in names} for _ in range(K)]
    for d_ in fev:   # create the events (torch creates them lazily on the first record)
        for ev in d_.values():
            ev.record(stream)
    barrier()
    n_keep = R.launches
    for i in range(K):
        flush(i & 0xFF)
        # keep the GPU busy (~50 us, outside the event pairs) while the host enqueues the
        # step, so no host-side gap falls between f0 and the forward kernel it brackets
        torch.cuda._sleep(100000)
        R.step(fev[i])
    barrier()
    R.launches = n_keep
    fwd_ms = [fev[i]["f0"].elapsed_time(fev[i]["f1"]) for i in range(K)]
    k2_ms = [fev[i]["k2a"].elapsed_time(fev[i]["k2b"]) for i in range(K)]
    k3_ms = [fev[i]["k3a"].elapsed_time(fev[i]["k3b"]) for i in range(K)]

    # ---- end to end through the public API with host buffers: every step uploads its
    # x and dY from pinned host memory and reads back y, dX, dA and dB.  Double-buffered
    # (one CUDA graph per buffer set): step i+1's upload and step i-1's read-back run on
    # copy streams while step i computes; all copies are inside the timed region.
    xs0 = R.distinct_x(0)
    old_aff = os.sched_getaffinity(0)
    local = gpu_local_cpus(local_rank)
    if local:   # pinned host buffers on the GPU's own NUMA node
        os.sched_setaffinity(0, local)
    try:
        hx = [t.cpu().pin_memory() for t in xs0]
        hdy = [e["dy_sets"][0].cpu().pin_memory() for e in lin]
        hy = [torch.empty(e["y_sets"][0].shape, dtype=torch.bfloat16).pin_memory() for e in lin]
        hdx = [torch.empty(e["dx_sets"][0].shape, dtype=torch.bfloat16).pin_memory() for e in lin]
        hda = [torch.empty(e["da"].shape, dtype=torch.float32).pin_memory() for e in lin]
        hdb = [torch.empty(e["db"].shape, dtype=torch.float32).pin_memory() for e in lin]
    finally:
        if local:
            os.sched_setaffinity(0, old_aff)
    h2d = sum(t.numel() * t.element_size() for t in hx + hdy)
    d2h = sum(t.numel() * t.element_size() for t in hy + hdx + hda + hdb)
    graphs = None
    if graph is not None:
        try:
            graphs = [graph, R.capture(1)[0]]
        except Exception as ex:
            print(f"bench: e2e graph capture failed ({ex!r}); e2e runs eager steps", file=sys.stderr)
            graphs = None
    up = torch.cuda.Stream(device=dev)
    down = torch.cuda.Stream(device=dev)
    xsets = [R.distinct_x(k) for k in range(2)]
    dsets = [[e["dy_sets"][k] for e in lin] for k in range(2)]

    def e2e_run(n_steps):
        uploaded = [torch.cuda.Event(), torch.cuda.Event()]
        computed = [torch.cuda.Event(), torch.cuda.Event()]
        drained = [torch.cuda.Event(), torch.cuda.Event()]
        start = torch.cuda.Event()
        start.record(stream)
        up.wait_event(start)
        down.wait_event(start)

        def upload(k):
            with torch.cuda.stream(up):
                for dst, src in zip(xsets[k], hx):
                    dst.copy_(src, non_blocking=True)
                for dst, src in zip(dsets[k], hdy):
                    dst.copy_(src, non_blocking=True)
                uploaded[k].record(up)

        upload(0)
        for it in range(n_steps):
            k = it % 2
            stream.wait_event(uploaded[k])
            if it >= 2:
                stream.wait_event(drained[k])   # step it-2's outputs in set k are read back
            if graphs is not None:
                graphs[k].replay()
            else:
                R.use_set(k)
                R.step()
            computed[k].record(stream)
            with torch.cuda.stream(down):
                down.wait_event(computed[k])
                for e, a_, b_, c_, d_ in zip(lin, hy, hdx, hda, hdb):
                    a_.copy_(e["y_sets"][k], non_blocking=True)
                    b_.copy_(e["dx_sets"][k], non_blocking=True)
                    c_.copy_(e["da_sets"][k], non_blocking=True)
                    d_.copy_(e["db_sets"][k], non_blocking=True)
                drained[k].record(down)
            if it + 1 < n_steps:
                if it >= 1:
                    up.wait_event(computed[1 - k])   # step it-1 no longer reads set 1-k
                upload(1 - k)
        stream.wait_stream(down)
        stream.wait_stream(up)

    e2e_run(3)
    barrier()
    Ke = max(3, min(K, 50))
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    e2e_run(Ke)
    s1.record(stream)
    barrier()
    R.use_set(0)
    e2e_ms = s0.elapsed_time(s1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- the HBM-bound kernels of the path, timed alone (report them in
    # GB/s against the measured HBM bandwidth): K4 merge of the first linear, the
    # gradient-only backward and one Adam step over every adapter -- L2 flushed before each
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
                flush(1)
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
        ad = []
        for e2 in lin:
            for t, g in ((e2["a"], e2["da"]), (e2["b"], e2["db"])):
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
        # the achievable HBM rate at each kernel's size: a plain device copy (torch copy_)
        # moving the same bytes (half read, half written), timed the same way -- MEASURED_PEAKS'
        # hbm_gbs is a 2 GiB copy; at tens of MB the launch ramp and drain cost a few us
        cp_src = torch.empty(max(merge_bytes, grads_bytes, adam_bytes) // 4 + 64, dtype=torch.float16, device=dev)
        cp_dst = torch.empty_like(cp_src)

        def copy_ref(nbytes):
            k = nbytes // 4
            t = timed(lambda: cp_dst[:k].copy_(cp_src[:k]))
            return {"us": t * 1e6, "gbs": 4 * k / t / 1e9}

        aux = {"merge": {"us": t_merge * 1e6, "bytes": merge_bytes, "gbs": merge_bytes / t_merge / 1e9,
                         "engine": "tcgen05 (B A in TMEM) + TMA load / store" if r0 % 8 == 0 and r0 <= 64
                         else "CUDA cores", "same_bytes_copy": copy_ref(merge_bytes)},
               "adam_all_adapters": {"us": t_adam * 1e6, "bytes": adam_bytes, "gbs": adam_bytes / t_adam / 1e9,
                                     "tensors": len(ad), "same_bytes_copy": copy_ref(adam_bytes)},
               "grads_only": {"us": t_grads * 1e6, "bytes": grads_bytes, "gbs": grads_bytes / t_grads / 1e9,
                              "kernels": "lora_linear_bwd with dx = NULL (gh row projection, K3)",
                              "same_bytes_copy": copy_ref(grads_bytes)}}

    # ---- report (rank 0)
    if rank == 0:
        peaks, peak_src = load_peaks()
        flops_step = workload_flops(wl)
        value = flops_step * K / (total_ms * 1e-3) / 1e12
        tokens = wl.linears[0].T
        l0 = wl.linears[0]
        grouped = bool(R.use_groups or R.tp_groups) and bool(wl.groups)
        roof_linears = [lin[i]["l"] for i in wl.groups[0]] if grouped else [l0]
        f_fwd = sum(fwd_flops(l) for l in roof_linears) / world
        f_dx = sum(bwd_dx_flops(l) for l in roof_linears) / world
        fwd_avg_s = float(np.mean(fwd_ms)) * 1e-3
        k2_avg_s = float(np.mean(k2_ms)) * 1e-3
        k3_avg_s = float(np.mean(k3_ms)) * 1e-3
        achieved = f_fwd / fwd_avg_s / 1e12
        peak = peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])
        hbm = peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"])
        traffic = None
        tp_path = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp_path):
            tj = json.load(open(tp_path))
            traffic = (tj.get("grouped_fwd_bytes_per_launch", {}).get(wl.key) if R.use_groups
                       else tj.get("fused_fwd_bytes_per_launch_single"))
        # K3 algorithmic bytes: every activation it reduces over read once (x once per
        # group sharing it, dY per linear) -- SURVEY.md 8(d) "K3" row without the tiny coefficients
        k3_lin = roof_linears
        k3_bytes = (2 * tokens * k3_lin[0].n + sum(2 * tokens * l.m for l in k3_lin)) / world
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cval, cdt, Rt, thr = cpu_oracle_sample(wl, target_s=args.cpu_seconds)
            cpu = {"value": cval / 1e12, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
                   "cpu_model": cpu_model_name(),
                   "sample": f"first {Rt} of {tokens} tokens of every linear of {wl.key} (complete "
                             f"{Rt}-token fwd+bwd problems), fp64 C oracle, {cdt:.1f} s"}
        line = {
            "metric": METRIC,
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl.key, "description": wl.description,
                       "linears": [f"{l.name}:{l.n}->{l.m}" for l in wl.linears],
                       "tokens": tokens, "rank": l0.r, "alpha": l0.alpha,
                       "global_batch": 1, "seq_len": tokens,
                       "parallelism": f"tp{world}" if comm is not None else "single",
                       "tp_comm": (("fused into the GEMMs over peer memory (lora_symm), reducer "
                                    + str(R.symm.last_placement) if args.comm == "fused"
                                    else "NCCL all-reduce after the GEMMs") if comm is not None else None),
                       "cuda_graph": graph is not None,
                       "grouped_calls": ([[wl.linears[i].name for i in g] for g in wl.groups] if grouped else None),
                       "shared_inputs": [[wl.linears[i].name for i in g] for g in wl.groups if len(g) > 1],
                       "lora_dropout": args.dropout,
                       "dropout_mask": (None if args.dropout == 0.0 else
                                        "kept: the forward stores the keep bits (T n / 8 bytes per linear) and "
                                        "M . x (2 T n bytes), the backward reads them" if args.dropout_mask == "kept" else
                                        "redrawn: the backward regenerates the Philox mask"),
                       "l2": "flushed between timed steps (2xL2 write then 2xL2 read, outside the "
                             "event pairs)"},
            "tokens_per_s": tokens * K / (total_ms * 1e-3),
            "pct_of_bf16_peak": value / (peak * world) * 100.0,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": (f"lora_linear_fwd_grouped of {[l.name for l in roof_linears]} (one fused K1 "
                                    f"launch{' + the dropout K0 launch before it' if args.dropout > 0 else ''}) "
                                    f"inside the step, " if len(roof_linears) > 1 else
                                    f"lora_linear_fwd of '{l0.name}' (fused K1"
                                    f"{' + dropout K0' if args.dropout > 0 else ''}) inside the step, ") +
                                   f"{f_fwd / 1e9:.2f} algorithmic GFLOP per launch, avg {fwd_avg_s * 1e6:.1f} us",
                         "peak_source": peak_src + " bf16_tflops (burst)",
                         # the same kernel against the sustained figure (cuBLAS back to back for 4 s):
                         # the fair denominator once a run lasts seconds and the 1 kW cap lowers clocks
                         "frac_of_sustained": (achieved / peaks["bf16_tflops_sustained"]
                                               if "bf16_tflops_sustained" in peaks else None),
                         "traffic_source": "ncu --set full dram__bytes_read+write of this launch "
                                           "(profiles/traffic.json, committed capture)"},
            "kernels_in_step": {
                "K1_fwd": {"us": fwd_avg_s * 1e6, "gflop": f_fwd / 1e9, "tflops": achieved,
                           "frac_of_peak": achieved / peak,
                           "us_median": float(np.median(fwd_ms)) * 1e3, "us_min": float(np.min(fwd_ms)) * 1e3,
                           "us_max": float(np.max(fwd_ms)) * 1e3},
                "K2_dx": {"us": k2_avg_s * 1e6, "gflop": f_dx / 1e9, "tflops": f_dx / k2_avg_s / 1e12,
                          "frac_of_peak": f_dx / k2_avg_s / 1e12 / peak,
                          "us_median": float(np.median(k2_ms)) * 1e3},
                "K3_dA_dB": {"us": k3_avg_s * 1e6, "bytes": k3_bytes, "gbs": k3_bytes / k3_avg_s / 1e9,
                             "frac_of_hbm": k3_bytes / k3_avg_s / 1e9 / hbm,
                             # in the graph-replayed step K3 starts in K2's last wave: what it adds
                             # to the step is the median step minus the K1 and K2 times (one group)
                             "exposed_in_step_us": ((float(np.median(step_ms)) * 1e3 - (fwd_avg_s + k2_avg_s) * 1e6)
                                                    if len(wl.groups) <= 1 and world == 1 else None),
                             "note": "event pair around the K3 launch, incl. its launch, setup and teardown; its "
                                     "token split is the step's (S = 1 at cfg2: 96 one-CTA jobs sized to start "
                                     "on the SMs K2's last wave frees), so the figure is not K3's standalone rate; "
                                     "per-phase probe in DESIGN.md 'K3 timings reconciled'"},
                "what": "first group's kernels, CUDA events on the launching stream inside K eager steps "
                        "(L2 flushed); K2/K3 via lora_profile_next_bwd, so K3 runs after K2 instead of in "
                        "its last wave"},
            "step_ms_median": float(np.median(step_ms)),
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": {"value": flops_step * Ke / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "what": "public API, per step: H2D x, dY from pinned host; D2H y, dX, dA, dB; "
                            "double-buffered, one CUDA graph per buffer set" if graphs else
                            "public API, eager steps; H2D x, dY; D2H y, dX, dA, dB"},
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
        if aux:
            for v in aux.values():
                v["frac_of_hbm"] = v["gbs"] / hbm
                if "same_bytes_copy" in v:
                    v["frac_of_same_bytes_copy"] = v["gbs"] / v["same_bytes_copy"]["gbs"]
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
    ap.add_argument("--config", default=None, choices=sorted(WORKLOADS),
                    help="workload (default: cfg2 at N = 1, cfg3 -- the sharded 7B layer set -- at N > 1)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed outputs")
    ap.add_argument("--force-tp", action="store_true",
                    help="run the tensor-parallel code path (NCCL communicator, TP entry points) even at N = 1")
    ap.add_argument("--dropout", type=float, default=0.0,
                    help="LoRA dropout p (Listing 3 LORA_DROPOUT = 0.05); 0 = the north-star path")
    ap.add_argument("--dropout-mask", choices=("kept", "redraw"), default="kept",
                    help="with --dropout: keep the forward's mask bits for the backward (lora_dropout.keep_bits) "
                         "or redraw them")
    ap.add_argument("--no-group", action="store_true",
                    help="one call per linear instead of grouped calls for linears sharing an input")
    ap.add_argument("--layer", choices=sorted(LAYERS), default=None,
                    help="time the Llama-2 decoder-layer train step (SURVEY 8(f) N4) instead of the LoRA linears")
    ap.add_argument("--comm", choices=["nccl", "fused"], default="nccl",
                    help="TP activation all-reduces: NCCL calls after the GEMMs, or fused into the GEMMs over "
                         "peer memory (lora_symm, SURVEY 8(f) N2)")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each step as one CUDA graph (auto: at every N, eager if capture fails)")
    args = ap.parse_args()
    if args.layer:   # the decoder-layer workload
        return run_layer(args, args.layer)
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    cfg = args.config or ("cfg2" if world == 1 else "cfg3")
    wl = WORKLOADS[cfg]
    if args.impl == "reference":
        return run_reference(args, wl)
    return run_ours(args, wl)


if __name__ == "__main__":
    sys.exit(main())

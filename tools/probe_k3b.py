"""K3 timing reconciliation (experiment, not product/tests): cfg2 q+v grouped
backward; CUDA events around K3 (lora_profile_next_bwd) next to the per-CTA
globaltimer stamps of a LORA_PROBE_K3 build, for several token splits S.

    python tools/probe_k3.py build          # builds build/probe/liblora_k3probe.so
    LORA_LIB_PATH=build/probe/liblora_k3probe.so python tools/probe_k3b.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402


def tod(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def setup(T, n, ms, r):
    x = None
    probs = []
    for i, m in enumerate(ms):
        d = make_lora_inputs(T, n, m, r, seed=10 + i)
        if x is None:
            x = tod(d["x"])
        w0, a, b, dy = (tod(d[k]) for k in ("w0", "a", "b", "dy"))
        y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
        probs.append((x, w0, a, b, dy, h))
    outs = [(torch.empty((T, n), dtype=torch.bfloat16, device="cuda"), torch.zeros((r, n), device="cuda"),
             torch.zeros((p[1].shape[0], r), device="cuda")) for p in probs]
    return probs, outs


def run(T, n, ms, r, want_dx=True, iters=12):
    probs, outs = setup(T, n, ms, r)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    flush_r = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    fn = getattr(L.lib, "lora_probe_k3_read", None)
    NS = 16384 * 6 + 2
    buf = (ctypes.c_ulonglong * NS)()
    if fn is not None:
        fn(buf, NS)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:   # (torch creates the CUDA event lazily, on its first record)
        e.record()
    rows = []
    for it in range(iters):
        flush.fill_(float(it))
        torch.sum(flush_r)   # (read pass: L2 left clean)
        torch.cuda.synchronize()
        L.lora_profile_next_bwd(*ev)
        o = outs if want_dx else [(None, a, b) for (_, a, b) in outs]
        L.lora_linear_bwd_grouped(probs, [16.0] * len(probs), outs=o, want_dx=want_dx)
        torch.cuda.synchronize()
        k3 = ev[2].elapsed_time(ev[3]) * 1e3
        k2 = ev[0].elapsed_time(ev[1]) * 1e3 if want_dx else 0.0
        rec = {"k3_event_us": k3, "k2_event_us": k2}
        if fn is not None:
            fn(buf, NS)
            allv = np.array(buf, dtype=np.uint64).astype(np.int64)
            pre, post = allv[-2], allv[-1]
            v = allv[:-2].reshape(-1, 6)
            v = v[v[:, 0] > 0]
            if len(v):
                t0 = v[:, 0].min()
                rec.update(ctas=len(v), pre_to_entry_us=(t0 - pre) / 1e3, span_us=(v[:, 5].max() - t0) / 1e3,
                           exit_to_post_us=(post - v[:, 5].max()) / 1e3,
                           start_spread_us=(v[:, 0].max() - t0) / 1e3,
                           setup_med_us=float(np.median(v[:, 1] - v[:, 0])) / 1e3,
                           main_med_us=float(np.median(v[:, 2] - v[:, 1])) / 1e3,
                           main_max_us=float((v[:, 2] - v[:, 1]).max()) / 1e3,
                           epi_med_us=float(np.median(v[:, 3] - v[:, 2])) / 1e3,
                           red_med_us=float(np.median(v[:, 4] - v[:, 3])) / 1e3,
                           exit_med_us=float(np.median(v[:, 5] - v[:, 4])) / 1e3)
        if it >= 3:
            rows.append(rec)
    keys = rows[0].keys()
    return {k: round(float(np.median([r_[k] for r_ in rows])), 2) for k in keys}


if __name__ == "__main__":
    shapes = {"cfg2_qv": (2048, 4096, [4096, 4096], 8), "cfg3_qkv": (4096, 4096, [4096] * 3, 16)}
    for S in os.environ.get("SWEEP_S", "auto,1,2").split(","):
        if S == "auto":
            os.environ.pop("LORA_K3_S", None)
        else:
            os.environ["LORA_K3_S"] = S
        for nm, sh in shapes.items():
            for wdx in (True, False):
                r = run(*sh, want_dx=wdx)
                print(json.dumps({"shape": nm, "S": S, "dx": wdx, **r}), flush=True)

"""K2 -> K3 overlap probe (cfg2 q + v grouped backward, x shared).

Times the grouped backward (one K2 launch + one K3 launch) replayed as a CUDA
graph, L2 flushed between replays, and -- for reference -- K2 alone (dA, dB not
requested).  Run twice, with LORA_K3_OVERLAP=0 and =1, and compare.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


T, n, m, r, alpha = 2048, 4096, 4096, 8, 16.0
dq, dv = make_lora_inputs(T, n, m, r, seed=1), make_lora_inputs(T, n, m, r, seed=2)
x = dev(dq["x"])
P = []
for d in (dq, dv):
    w0, a, b, dy = (dev(d[k]) for k in ("w0", "a", "b", "dy"))
    _, h = L.lora_linear_fwd(x, w0, a, b, alpha)
    P.append((x, w0, a, b, dy, h))
outs = [(torch.empty((T, n), dtype=torch.bfloat16, device="cuda"), torch.empty((r, n), device="cuda"),
         torch.empty((m, r), device="cuda")) for _ in P]
outs_dx = [(o[0], None, None) for o in outs]
ws = torch.empty(1 << 26, dtype=torch.uint8, device="cuda")
flush_w = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
flush_r = torch.zeros_like(flush_w)
s = torch.cuda.Stream()


def graph_of(fn):
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g


def full():
    L.lora_linear_bwd_grouped(P, [alpha, alpha], outs=outs, workspace=ws, stream=s)


def dx_only():
    probs = [(px, pw, pa, pb, pdy, ph) for (px, pw, pa, pb, pdy, ph) in P]
    for (dxo, _, _), pr in zip(outs, probs):
        L.lora_linear_bwd(pr[0], pr[1], pr[2], pr[3], pr[4], alpha, h_saved=pr[5], dx=dxo, want_da=False,
                          want_db=False, workspace=ws, stream=s)


for name, fn in (("k2+k3 grouped", full), ("k2 only (2 calls)", dx_only)):
    g = graph_of(fn)
    ts = []
    for i in range(300):
        with torch.cuda.stream(s):
            flush_w.fill_(float(i))
            torch.sum(flush_r)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        if i >= 20:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"LORA_K3_OVERLAP={os.environ.get('LORA_K3_OVERLAP', '1')} {name}: median {np.median(ts):.1f} us "
          f"p10 {np.percentile(ts, 10):.1f} p90 {np.percentile(ts, 90):.1f}")

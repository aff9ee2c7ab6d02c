"""Times lora_merge (K4) at the workloads' projection shapes.

Two protocols: (a) one call per event pair after an L2 flush that writes then
reads 2x L2 (clean L2, as bench.py); (b) 20 back-to-back calls over 4 rotating
W0 / W' buffer sets (working set > L2), average per call -- no launch gaps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402

dev = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()  # noqa: E731
flush = torch.empty(64 << 20, device="cuda")
for (m, n, r) in ((4096, 4096, 8), (11008, 4096, 16), (4096, 11008, 16), (28672, 8192, 16), (4096, 4096, 64)):
    d = make_lora_inputs(16, n, m, r, seed=1)
    w0, a, b = (dev(d[k]) for k in ("w0", "a", "b"))
    sets = [(w0.clone(), torch.empty_like(w0)) for _ in range(4)]
    out = torch.empty_like(w0)
    ts = []
    for i in range(25):
        flush.fill_(i)
        float(flush[:1024].sum())   # (clean L2: the read evicts the dirty lines)
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lora_merge(w0, a, b, 16.0, w_out=out)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    byts = 4 * m * n + 2 * r * (m + n)
    for k in range(8):
        L.lora_merge(sets[k % 4][0], a, b, 16.0, w_out=sets[k % 4][1])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.fill_(0)
    e0.record()
    for k in range(20):
        L.lora_merge(sets[k % 4][0], a, b, 16.0, w_out=sets[k % 4][1])
    e1.record()
    torch.cuda.synchronize()
    us2 = e0.elapsed_time(e1) * 1e3 / 20
    # the same bytes as a plain device copy (torch copy_ of W0 -> W'): the achievable
    # read + write rate at this size, next to the 1 GiB-copy peak of MEASURED_PEAKS
    for k in range(8):
        sets[k % 4][1].copy_(sets[k % 4][0])
    e0.record()
    for k in range(20):
        sets[k % 4][1].copy_(sets[k % 4][0])
    e1.record()
    torch.cuda.synchronize()
    us3 = e0.elapsed_time(e1) * 1e3 / 20
    print(f"{os.environ.get('TAG', '')} merge {m}x{n} r{r}: single {us:.1f} us {byts / us / 1e3:.0f} GB/s | "
          f"back-to-back {us2:.1f} us {byts / us2 / 1e3:.0f} GB/s | copy_ {us3:.1f} us {4 * m * n / us3 / 1e3:.0f} GB/s")

"""Times lora_merge (K4) at cfg2 / cfg5 shapes, L2 flushed before each call."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402

dev = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()  # noqa: E731
flush = torch.empty(64 << 20, device="cuda")
for (m, n, r) in ((4096, 4096, 8), (28672, 8192, 16)):
    d = make_lora_inputs(16, n, m, r, seed=1)
    w0, a, b = (dev(d[k]) for k in ("w0", "a", "b"))
    out = torch.empty_like(w0)
    ts = []
    for i in range(25):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lora_merge(w0, a, b, 16.0, w_out=out)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    byts = 4 * m * n + 2 * r * (m + n)
    print(f"{os.environ.get('TAG', '')} merge {m}x{n} r{r}: {us:.1f} us, {byts / us / 1e3:.0f} GB/s")

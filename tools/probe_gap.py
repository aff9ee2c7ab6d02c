"""Host-gap reconciliation (experiment, not product/tests): time the same
library call (a) eagerly between two events, (b) eagerly behind a GPU sleep
kernel so the launches are queued before the first event fires, (c) as a CUDA
graph replay behind the sleep.  cfg2 'q' shapes, L2 flushed before each."""
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


d = make_lora_inputs(2048, 4096, 4096, 8, seed=2403)
x, w0, a, b, dy = (tod(d[k]) for k in ("x", "w0", "a", "b", "dy"))
y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
w_out = torch.empty_like(w0)
da, db = torch.zeros((8, 4096), device="cuda"), torch.zeros((4096, 8), device="cuda")
flushbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()


def timed(fn, mode, reps=20):
    s = torch.cuda.current_stream()
    g = None
    if mode == "graph":
        with torch.cuda.stream(side):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            fn()
        torch.cuda.synchronize()
    for _ in range(3):
        g.replay() if g else fn()
    ts = []
    for _ in range(reps):
        flushbuf.fill_(1)
        if mode != "eager":
            torch.cuda._sleep(200000)   # ~100 us: the host queues fn before a0 fires
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s)
        g.replay() if g else fn()
        a1.record(s)
        torch.cuda.synchronize()
        ts.append(a0.elapsed_time(a1) * 1e3)
    return round(float(np.median(ts)), 2)


fns = {
    "merge": lambda: L.lora_merge(w0, a, b, 16.0, w_out=w_out, stream=torch.cuda.current_stream()),
    "grads_only": lambda: L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_dx=False, da=da, db=db,
                                            stream=torch.cuda.current_stream()),
    "copy_64MB": lambda: w_out.copy_(w0),
}
for nm, fn in fns.items():
    print(json.dumps({"fn": nm, **{m: timed(fn, m) for m in ("eager", "eager_sleep", "graph")}}), flush=True)

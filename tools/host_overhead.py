"""Host-side cost per C-ABI call (eager, no graph): wall time of N back-to-back
calls on tiny shapes, where the GPU work is negligible."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402


def dev(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()


d = make_lora_inputs(256, 256, 256, 8, seed=1)
x, w0, a, b, dy = (dev(d[k]) for k in ("x", "w0", "a", "b", "dy"))
y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
dx, da, db = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h)
wsf = torch.empty(L.lora_linear_fwd_workspace_bytes(L.dims(256, 256, 256, 8, 16.0)), dtype=torch.uint8, device="cuda")
wsb = torch.empty(L.lora_linear_bwd_workspace_bytes(L.dims(256, 256, 256, 8, 16.0)), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for name, fn in (("fwd", lambda: L.lora_linear_fwd(x, w0, a, b, 16.0, y=y, h_out=h, workspace=wsf, stream=s)),
                 ("bwd", lambda: L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dx=dx, da=da, db=db,
                                                   workspace=wsb, stream=s))):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    n = 500
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host {1e6 * (t1 - t0) / n:.1f} us/call, end-to-end {1e6 * (t2 - t0) / n:.1f} us/call")

# the C call alone (arguments prepared once): what the library itself costs per call
import ctypes  # noqa: E402
dd = L.dims(256, 256, 256, 8, 16.0)
args = (ctypes.byref(dd), x.data_ptr(), w0.data_ptr(), a.data_ptr(), b.data_ptr(), None, y.data_ptr(), h.data_ptr(),
        wsf.data_ptr(), wsf.numel(), s.cuda_stream)
for _ in range(20):
    L.lib.lora_linear_fwd(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500):
    L.lib.lora_linear_fwd(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"fwd C call only: {1e6 * (t1 - t0) / 500:.1f} us/call")

"""ncu target for the HBM-bound side kernels at cfg2 'q': K4 merge and the
dX-free backward (B^T pack + h split, gh row projection + split, K3)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402

dev = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()  # noqa: E731
d = make_lora_inputs(2048, 4096, 4096, 8, seed=2403)
x, w0, a, b, dy = (dev(d[k]) for k in ("x", "w0", "a", "b", "dy"))
_, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
out = torch.empty_like(w0)
flush = torch.empty(64 << 20, device="cuda")
for i in range(3):
    flush.fill_(i)
    L.lora_merge(w0, a, b, 16.0, w_out=out)
    flush.fill_(i)
    L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_dx=False)
torch.cuda.synchronize()

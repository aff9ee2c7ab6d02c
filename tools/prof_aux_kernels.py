"""ncu helper: the CUDA-core kernels (merge, dropout K0, Adam) at cfg2 shapes."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402

d = make_lora_inputs(2048, 4096, 4096, 8, seed=2403)


def dev(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()


x, w0, a, b, dy = (dev(d[k]) for k in ("x", "w0", "a", "b", "dy"))
L.lora_merge(w0, a, b, 16.0)
y, h = L.lora_linear_fwd(x, w0, a, b, 16.0, dropout=(0.05, 1, 0))
L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dropout=(0.05, 1, 0))
ts = [(a.clone(), torch.randn(a.shape, device="cuda"), torch.zeros(a.shape, device="cuda"),
       torch.zeros(a.shape, device="cuda"), a.float()),
      (b.clone(), torch.randn(b.shape, device="cuda"), torch.zeros(b.shape, device="cuda"),
       torch.zeros(b.shape, device="cuda"), b.float())]
L.lora_adam_step(ts, 1, 1e-3)
torch.cuda.synchronize()

import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2403_11366_b200 as L
from synth import make_lora_inputs
d = make_lora_inputs(2048, 4096, 4096, 8, seed=2403)
dev = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()
x, w0, a, b, dy = (dev(d[k]) for k in ("x", "w0", "a", "b", "dy"))
for _ in range(3):
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h)
torch.cuda.synchronize()

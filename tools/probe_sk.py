"""Stream-K timeline probe: builds liblora with -DLORA_PROBE_SK (every unit's
epilogue prints its MMA-done and end times, ns from kernel start) and runs ONE
dX launch (cfg2 q, dA/dB skipped) and one forward.
    python tools/probe_sk.py build   (CPU host)   /   python tools/probe_sk.py run   (GPU)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "build", "probe", "liblora_sk.so")

if sys.argv[1] == "build":
    import importlib.util
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2403_11366_b200", "build.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    m.build(force=True, out=LIB, defines=("LORA_PROBE_SK",))
    sys.exit(0)

os.environ["LORA_LIB_PATH"] = LIB
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2403_11366_b200 as L  # noqa: E402
from synth import make_lora_inputs  # noqa: E402

d = make_lora_inputs(2048, 4096, 4096, 8, seed=1)
dev = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()  # noqa: E731
x, w0, a, b, dy = (dev(d[k]) for k in ("x", "w0", "a", "b", "dy"))
mode = sys.argv[2] if len(sys.argv) > 2 else "dx"
import ctypes  # noqa: E402
buf = (ctypes.c_ulonglong * (4 * 4096))()
for it in range(3):
    if mode == "dx":
        L.lora_linear_bwd(x, w0, a, b, dy, 16.0, want_da=False, want_db=False)
    elif mode == "dxdrop":
        L.lora_linear_bwd(x, w0, a, b, dy, 16.0, want_da=False, want_db=False, dropout=(0.05, 1, 2))
    else:
        L.lora_linear_fwd(x, w0, a, b, 16.0)
    torch.cuda.synchronize()
    n = L.lib.lora_probe_sk_dump(buf, 4096)
    if it < 2:
        continue
    rows = []
    for i in range(n):
        r0, r1, t0, t1 = buf[4 * i: 4 * i + 4]
        rows.append((r0 >> 32, (r0 >> 8) & 0xFFFFFF, r0 & 0xFF, r1 >> 32, r1 & 0xFFFFFFFF, t0 / 1e3, t1 / 1e3))
    rows.sort()
    ends = {}
    for r in rows:
        ends[r[0]] = max(ends.get(r[0], 0), r[6])
    print(f"{mode} LORA_STREAMK={os.environ.get('LORA_STREAMK', '1')}: units {len(rows)} "
          f"max end {max(ends.values()):.1f} us, min end {min(ends.values()):.1f} us")
    epi = [r[6] - r[5] for r in rows]
    print(f"epilogue (end - mma_done) us: median {np.median(epi):.2f} max {max(epi):.2f}")
    for r in rows[:40]:
        print("pair %3d unit %d role %d kb %3d-%3d mma_done %7.1f end %7.1f" % r)

"""Kernel experiments (not part of the product or the tests).

Times the fused forward (K1) and the dX kernel (K2, called with dA/dB skipped)
at cfg2 shapes for several compile-time variants of liblora.so, each loaded
in its own subprocess through LORA_LIB_PATH.

    python tools/probe_gemm.py build        # on the CPU host: build variants into build/probe/
    python tools/probe_gemm.py run          # on the GPU: time every variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "probe")

VARIANTS = {
    "base": (),
    "stages3": ("LORA_STAGES_CAP=3",),
    "stages2": ("LORA_STAGES_CAP=2",),
    "no_tail": ("LORA_PROBE_NO_TAIL",),
    "no_store": ("LORA_PROBE_NO_STORE",),
}
EXTRA = json.loads(os.environ.get("PROBE_VARIANTS", "{}"))
VARIANTS.update({k: tuple(v) for k, v in EXTRA.items()})


def build():
    import __graft_entry__
    b = __graft_entry__._build_module()
    os.makedirs(OUT, exist_ok=True)
    for name, defs in VARIANTS.items():
        b.build(out=os.path.join(OUT, f"liblora_{name}.so"), defines=defs)
        print("built", name, flush=True)


def time_one(T=2048, n=4096, m=4096, r=8, iters=50):
    import numpy as np
    import torch

    import paper_2403_11366_b200 as L
    from synth import make_lora_inputs
    d = make_lora_inputs(T, n, m, r, seed=2403)

    def dev(bits):
        return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()

    x, w0, a, b, dy = (dev(d[k]) for k in ("x", "w0", "a", "b", "dy"))
    y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
    dx, _, _ = L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_da=False, want_db=False)
    flush_w = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    flush_r = torch.zeros_like(flush_w)

    class _Flush:  # write 256 MiB, then read 256 MiB: cold L2 without dirty lines
        def fill_(self, v):
            flush_w.fill_(float(v))
            torch.sum(flush_r)

    flush = _Flush()
    res = {}
    da = torch.zeros((r, n), device="cuda")
    db = torch.zeros((m, r), device="cuda")
    for name, fn in (("fwd", lambda: L.lora_linear_fwd(x, w0, a, b, 16.0, y=y, h_out=h)),
                     ("dx", lambda: L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, dx=dx,
                                                      want_da=False, want_db=False)),
                     ("grads_gh_k3", lambda: L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_dx=False,
                                                               da=da, db=db)),
                     ("db_k3_only", lambda: L.lora_linear_bwd(x, w0, a, b, dy, 16.0, h_saved=h, want_dx=False,
                                                              want_da=False, db=db)),
                     # references for a 16 MiB read of dY on this box / in this harness
                     ("torch_sum_dy", lambda: torch.sum(dy, dtype=torch.float32)),
                     ("torch_copy_dy", lambda: dx.copy_(dy)),
                     # cuBLAS on the same base GEMM shapes (context for the GEMM efficiency)
                     ("cublas_fwd_base", lambda: torch.matmul(x, w0.t(), out=y)),
                     ("cublas_dx_base", lambda: torch.matmul(dy, w0, out=dx))):
        for _ in range(5):
            fn()
        ts = []
        for _ in range(iters):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = float(np.median(ts))
        flops = 2 * T * m * n + 2 * T * r * (m + n)
        res[name] = {"us": us, "tflops": flops / us / 1e6}
    return res


def run():
    out = {}
    jobs = [(name, os.path.join(OUT, f"liblora_{name}.so"), {}) for name in VARIANTS]
    # the in-tree library with the CTA-pair choice forced either way
    tree = os.path.join(ROOT, "paper_2403_11366_b200", "liblora.so")
    jobs += [(f"tree_cg{cg}", tree, {"LORA_CTA_GROUP": str(cg)}) for cg in (1, 2)]
    jobs += [("tree_k3cluster", tree, {"LORA_K3": "cluster"})]
    for name, lib, extra in jobs:
        if not os.path.exists(lib):
            continue
        env = dict(os.environ, LORA_LIB_PATH=lib, **extra)
        p = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True,
                           timeout=300)
        try:
            out[name] = json.loads(p.stdout.strip().splitlines()[-1])
        except Exception:
            out[name] = {"error": (p.stderr or p.stdout)[-500:]}
        print(name, json.dumps(out[name]), flush=True)
    return out


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "run"
    if cmd == "build":
        build()
    elif cmd == "one":
        print(json.dumps(time_one()))
    else:
        run()

"""K3 (tensor-core dA / dB) experiments (not part of the product or the tests).

Builds liblora.so variants with per-CTA globaltimer stamps (LORA_PROBE_K3) and
runs the grouped backward of a q/k/v-style group (three linears reading the
SAME x) at cfg3 sizes, reporting per-CTA phase times of the K3 launch.

    python tools/probe_k3.py build      # CPU host
    python tools/probe_k3.py run        # GPU
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "probe")

VARIANTS = {
    "k3probe": ("LORA_PROBE_K3",),
    "k3one": ("LORA_PROBE_K3", "LORA_K3_ONE_PER_SM"),
    "k3st3": ("LORA_PROBE_K3", "LORA_K3_STAGES=3"),
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


def one(T, n, ms, r, iters=20):
    import ctypes

    import numpy as np
    import torch

    import paper_2403_11366_b200 as L
    from synth import make_lora_inputs
    dev = "cuda"

    def tod(bits):
        return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)

    x = None
    probs = []
    for i, m in enumerate(ms):
        d = make_lora_inputs(T, n, m, r, seed=10 + i)
        if x is None:
            x = tod(d["x"])
        w0, a, b, dy = (tod(d[k]) for k in ("w0", "a", "b", "dy"))
        y, h = L.lora_linear_fwd(x, w0, a, b, 16.0)
        probs.append((x, w0, a, b, dy, h))
    outs = [(torch.empty((T, n), dtype=torch.bfloat16, device=dev), torch.zeros((r, n), device=dev),
             torch.zeros((p[1].shape[0], r), device=dev)) for p in probs]
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    fn = getattr(L.lib, "lora_probe_k3_read", None)
    buf = (ctypes.c_ulonglong * (16384 * 4))()
    if fn is not None:
        fn(buf, 16384 * 4)   # clear stamps of earlier launches
    phases = []
    for it in range(iters):
        flush.fill_(float(it))
        torch.cuda.synchronize()
        L.lora_linear_bwd_grouped(probs, [16.0] * len(probs), outs=outs)
        torch.cuda.synchronize()
        if fn is not None and it < 3:
            fn(buf, 16384 * 4)
        if fn is not None and it >= 3:
            fn(buf, 16384 * 4)
            v = np.array(buf, dtype=np.uint64).reshape(-1, 4)
            v = v[v[:, 0] > 0].astype(np.int64)
            if len(v) == 0:
                continue
            t0 = v[:, 0].min()
            phases.append(dict(
                ctas=len(v),
                total_us=(v[:, 3].max() - t0) / 1e3,
                start_spread_us=(v[:, 0].max() - t0) / 1e3,
                main_us=float(np.median(v[:, 1] - v[:, 0])) / 1e3,
                main_max_us=float((v[:, 1] - v[:, 0]).max()) / 1e3,
                epi_us=float(np.median(v[:, 2] - v[:, 1])) / 1e3,
                red_us=float(np.median(v[:, 3] - v[:, 2])) / 1e3,
            ))
    if not phases:
        return {}
    keys = phases[0].keys()
    return {k: float(np.median([p[k] for p in phases])) for k in keys}


def run_variant(name):
    env = dict(os.environ, LORA_LIB_PATH=os.path.join(OUT, f"liblora_{name}.so"))
    code = ("import json, tools.probe_k3 as p; "
            "print(json.dumps({'qkv': p.one(4096, 4096, [4096, 4096, 4096], 16), "
            "'gateup': p.one(4096, 4096, [11008, 11008], 16), "
            "'cfg2_qv': p.one(2048, 4096, [4096, 4096], 8)}))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600)
    if out.returncode != 0:
        return {"error": out.stderr[-2000:]}
    return json.loads(out.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        names = sys.argv[2:] or list(VARIANTS)
        for nm in names:
            print(nm, json.dumps(run_variant(nm)), flush=True)

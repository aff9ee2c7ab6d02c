"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
the bench.

This module holds none of the method's arithmetic: it only draws random
numbers, rounds them to bf16 bit patterns (RNE), and names the workload shapes
of BASELINE.json.  Both sides (oracle/ and the CUDA path) consume the same
bit patterns.  Recipe ("Input recipe"):

  * numpy SeedSequence(seed).spawn(6) -> one PCG64 stream per tensor, in the
    fixed order x, W0, A, B, G(=dY), bias;
  * x, G ~ N(0, 1); W0, A ~ N(0, 1/n) (A: N(0, 1/d_in)); B ~ N(0, 1/r);
    bias ~ N(0, 1);  float32 normals rounded to nearest-even bf16.
  * B is never zero in perf runs; the B = 0 case of the
    paper's init is a separate, explicit test input.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_SEED = 2403


def f32_to_bf16_bits(a) -> np.ndarray:
    """Round float32 values to the nearest-even bf16 and return uint16 bits."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f64(bits) -> np.ndarray:
    """Widen bf16 bit patterns exactly to float64."""
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def bf16_bits_to_f32(bits) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


@dataclass(frozen=True)
class LoraShape:
    """One LoRA linear: T tokens, d_in = n, d_out = m, rank r, alpha."""
    name: str
    T: int
    n: int
    m: int
    r: int
    alpha: float


@dataclass(frozen=True)
class Workload:
    """A BASELINE.json config: a list of LoRA linears sharing T."""
    key: str
    description: str
    linears: tuple
    tp_modes: tuple  # per linear: "column" | "row" (PAPER.md:122 reading, R10)
    groups: tuple    # linears that take the same input in the model (q,k,v / gate,up / q,v)


def _wl(key, desc, T, r, alpha, specs):
    lin = tuple(LoraShape(nm, T, n, m, r, alpha) for nm, n, m, _ in specs)
    modes = tuple(md for _, _, _, md in specs)
    names = [nm for nm, _, _, _ in specs]
    shared = [("q", "k", "v"), ("gate", "up")]
    groups, seen = [], set()
    for i, nm in enumerate(names):
        if i in seen:
            continue
        g = [i]
        for s in shared:
            if nm in s:
                g = [j for j, nj in enumerate(names) if nj in s]
        seen.update(g)
        groups.append(tuple(g))
    return Workload(key, desc, lin, modes, tuple(groups))


# BASELINE.json "configs", in order.  alpha = 16 (Listing 3 default,
# PAPER.md:81) wherever the config line does not state it (R3).
WORKLOADS = {
    "cfg1": _wl("cfg1", "single LoRA linear 64->64, r=4, 128 tokens", 128, 4, 16.0,
                [("lin", 64, 64, "column")]),
    "cfg2": _wl("cfg2", "Llama-2-7B q/v projection 4096x4096, r=8, alpha=16, batch 1 x seq 2048",
                2048, 8, 16.0,
                [("q", 4096, 4096, "column"), ("v", 4096, 4096, "column")]),
    "cfg3": _wl("cfg3", "Llama-2-7B decoder-layer LoRA set, r=16, seq 4096", 4096, 16, 16.0,
                [("q", 4096, 4096, "column"), ("k", 4096, 4096, "column"),
                 ("v", 4096, 4096, "column"), ("o", 4096, 4096, "row"),
                 ("gate", 4096, 11008, "column"), ("up", 4096, 11008, "column"),
                 ("down", 11008, 4096, "row")]),
    "cfg4": _wl("cfg4", "Llama-2-13B decoder-layer LoRA set, r=8, seq 4096", 4096, 8, 16.0,
                [("q", 5120, 5120, "column"), ("k", 5120, 5120, "column"),
                 ("v", 5120, 5120, "column"), ("o", 5120, 5120, "row"),
                 ("gate", 5120, 13824, "column"), ("up", 5120, 13824, "column"),
                 ("down", 13824, 5120, "row")]),
    "cfg5": _wl("cfg5", "Llama-2-70B decoder-layer LoRA set (GQA kv 1024), r=16, seq 4096",
                4096, 16, 16.0,
                [("q", 8192, 8192, "column"), ("k", 8192, 1024, "column"),
                 ("v", 8192, 1024, "column"), ("o", 8192, 8192, "row"),
                 ("gate", 8192, 28672, "column"), ("up", 8192, 28672, "column"),
                 ("down", 28672, 8192, "row")]),
}


def make_lora_inputs(T, n, m, r, seed=DEFAULT_SEED, bias=False, zero_b=False,
                     dist="normal"):
    """Draw one LoRA linear's inputs as bf16 bit patterns (uint16 arrays).

    dist="normal"  : the parity/perf recipe in the module docstring.
    dist="ternary" : values in {-1, 0, 0, 1} (SURVEY.md 8(c) pin 5), so every
                     product and short sum is a small integer.
    Returns dict x[T,n], w0[m,n], a[r,n], b[m,r], dy[T,m], bias[m] or None.
    """
    ss = np.random.SeedSequence(seed).spawn(6)
    gens = [np.random.Generator(np.random.PCG64(s)) for s in ss]

    def draw(g, shape, std):
        if dist == "ternary":
            v = g.integers(0, 4, size=shape)
            return np.choose(v, [-1.0, 0.0, 0.0, 1.0]).astype(np.float32)
        return (g.standard_normal(size=shape, dtype=np.float32) * np.float32(std))

    out = {
        "x": f32_to_bf16_bits(draw(gens[0], (T, n), 1.0)),
        "w0": f32_to_bf16_bits(draw(gens[1], (m, n), 1.0 / np.sqrt(n))),
        "a": f32_to_bf16_bits(draw(gens[2], (r, n), 1.0 / np.sqrt(n))),
        "b": f32_to_bf16_bits(draw(gens[3], (m, r), 1.0 / np.sqrt(r))),
        "dy": f32_to_bf16_bits(draw(gens[4], (T, m), 1.0)),
        "bias": f32_to_bf16_bits(draw(gens[5], (m,), 1.0)) if bias else None,
    }
    if zero_b:
        out["b"] = np.zeros((m, r), np.uint16)
    return out


def algorithmic_flops(T, n, m, r) -> int:
    """fwd+bwd algorithmic FLOPs of one LoRA linear:
    4 T m n + 6 T r (m + n); no dW0 (frozen), no padding or recompute."""
    return 4 * T * m * n + 6 * T * r * (m + n)


def make_layer_inputs(T, d, f, heads, r, seed=DEFAULT_SEED):
    """Inputs of one Llama-2 decoder layer with LoRA on all seven projections
    (SURVEY.md 8(f) N4), as bf16 bit patterns: x, dout ~ N(0, 1); every W0 of
    shape [m, n] ~ N(0, 1/n); A ~ N(0, 1/n); B ~ N(0, r / 1024) (a trained
    adapter's delta is a fraction of the base projection: with h ~ N(0, 1) per
    rank index and s = 16 / r the delta's std is s sqrt(r) sqrt(r) / 32 = 1/2 of
    the base's at EVERY rank -- round 2 used N(0, 1/(16 r)), which is this at
    r = 8 only and made small-rank layers LoRA-dominated (std 4 at r = 1) with
    saturated attention scores; the single-linear recipe's N(0, 1/r) would do so
    at every rank); the RMSNorm weights g1, g2 ~ 1 + N(0, 0.1^2).  One PCG64
    stream per tensor, fixed order."""
    shapes = {"q": (d, d), "k": (d, d), "v": (d, d), "o": (d, d), "gate": (f, d), "up": (f, d), "down": (d, f)}
    streams = np.random.SeedSequence(seed).spawn(4 + 3 * len(shapes))
    rng = iter(np.random.Generator(np.random.PCG64(s)) for s in streams)
    out = {"x": f32_to_bf16_bits(next(rng).standard_normal((T, d), dtype=np.float32)),
           "dout": f32_to_bf16_bits(next(rng).standard_normal((T, d), dtype=np.float32)),
           "g1": f32_to_bf16_bits(1.0 + 0.1 * next(rng).standard_normal(d, dtype=np.float32)),
           "g2": f32_to_bf16_bits(1.0 + 0.1 * next(rng).standard_normal(d, dtype=np.float32))}
    for name, (m, n) in shapes.items():
        out["w0_" + name] = f32_to_bf16_bits(next(rng).standard_normal((m, n), dtype=np.float32) / np.sqrt(n))
        out["a_" + name] = f32_to_bf16_bits(next(rng).standard_normal((r, n), dtype=np.float32) / np.sqrt(n))
        out["b_" + name] = f32_to_bf16_bits(next(rng).standard_normal((m, r), dtype=np.float32) *
                                            np.float32(np.sqrt(r) / 32.0))
    return out

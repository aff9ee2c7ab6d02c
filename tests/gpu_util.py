"""Helpers for the GPU parity tests: move the shared bf16 bit patterns to the
device and compare the CUDA path against the fp64 oracle."""
import numpy as np
import torch


def dev_bf16(bits):
    """uint16 bf16 bit patterns -> CUDA bf16 tensor (same bits)."""
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    return torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).cuda()


def host_f64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def bits_of(t):
    """CUDA bf16 tensor -> uint16 numpy bit patterns."""
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def relF(gpu, ref):
    """Relative Frobenius error ||gpu - ref|| / ||ref|| in fp64;
    if ref is identically zero, gpu must be exactly zero."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    nr = np.linalg.norm(ref)
    if nr == 0.0:
        return 0.0 if np.all(gpu == 0.0) else float("inf")
    return float(np.linalg.norm(gpu - ref) / nr)


def rne_bf16_f64(v):
    """Round fp64 values to bf16 via fp32 (as a reference rounding)."""
    f = np.asarray(v, np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32) << 16
    return r.view(np.float32).astype(np.float64)


# Tolerances written from north_star (BASELINE.json): relative Frobenius error
# 1e-2 for outputs (y, dX), 2e-2 for gradients (dA, dB).
TOL_OUT = 1e-2
TOL_GRAD = 2e-2

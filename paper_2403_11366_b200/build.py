"""In-tree build of liblora.so (sm_100a) with nvcc.

    python -m paper_2403_11366_b200.build [--force]

Produces paper_2403_11366_b200/liblora.so next to this file.  The library is
statically linked against cudart; the driver API (cuTensorMapEncodeTiled) is
resolved at run time and NCCL is dlopen'ed by lora_comm_init, so the library
loads (and can be validated) on a machine without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "liblora.so")
SOURCES = ["lora_gemm.cu", "lora_grad.cu", "lora_grad_mma.cu", "lora_dropout.cu", "lora_aux.cu", "lora_merge_mma.cu", "lora_symm.cu", "lora_layer.cu", "lora_api.cpp", "lora_comm.cpp", "lora_export.cpp"]
HEADERS = ["sm100_ptx.cuh", "lora_philox.cuh", "lora_kernels.h", "lora_internal.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # noqa: F401  (pip wheel nvidia-nccl-cu12, same as torch's)
        base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) \
            else list(nvidia.nccl.__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except Exception:
        pass
    return "/usr/include"


def nccl_library() -> str | None:
    """Path of the NCCL shared library torch uses (for LORA_NCCL_LIB)."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        p = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    except Exception:
        pass
    return None


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "lora.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Build liblora.so (or, with `out`/`defines`, an experiment variant).

    Each source is compiled to an object in parallel (one nvcc per file), then
    linked; the objects live in a per-process scratch directory next to the
    library so concurrent builders never share a partial file."""
    import shutil
    import tempfile
    from concurrent.futures import ThreadPoolExecutor

    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    flags = [*ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3",
             "-I", INCLUDE, "-I", CSRC, "-I", _nccl_include(),
             "-DLORA_BUILD", *[f"-D{d}" for d in defines]]
    tmp = tempfile.mkdtemp(prefix=".build", dir=PKG)
    try:
        objs = [os.path.join(tmp, f + ".o") for f in SOURCES]

        def compile_one(i):
            subprocess.check_call([nvcc, *flags, "-c", "-o", objs[i], os.path.join(CSRC, SOURCES[i])])

        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
            list(ex.map(compile_one, range(len(SOURCES))))
        subprocess.check_call([nvcc, *ARCH, "-shared", "-o", f"{target}.tmp{os.getpid()}", *objs,
                               "-ldl", "-lpthread"])
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    os.replace(f"{target}.tmp{os.getpid()}", target)   # atomic: concurrent builders never see a partial file
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)

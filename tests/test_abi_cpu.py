"""C-ABI tests that need no GPU: the library loads, exports every symbol
include/lora.h declares, and validates its arguments synchronously (returning
the documented status before any CUDA call).  No compute is invoked here."""
import ctypes
import os

import pytest

import paper_2403_11366_b200 as L


def test_library_exports_every_header_symbol():
    names = L.header_functions()
    assert "lora_linear_fwd" in names and "lora_linear_bwd" in names and "lora_merge" in names
    missing = [n for n in names if not hasattr(L.lib, n)]
    assert not missing, f"liblora.so lacks {missing}"
    assert L.lib.lora_version() >= 100


def test_sass_is_sm100a_tensor_core_code():
    """The fused GEMMs must be tcgen05 (UTC*MMA) fed by TMA (UTMALDG).  Legacy
    mma.sync (HMMA) appears only in the dropout K0 (dropout_h_group_kernel: the
    rank-r product of the masked input, 2 T n r FLOPs beside its Philox draws;
    DESIGN.md dropout path) -- no GEMM of the path uses it."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", L.LIB_PATH], capture_output=True,
                                       text=True).stdout
    funcs = out.split("Function : ")
    with_hmma = [f.split()[0] for f in funcs[1:] if " HMMA" in f]
    assert with_hmma and all("dropout_h_group_kernel" in f for f in with_hmma), with_hmma


def test_status_strings():
    for code, name in L.STATUS.items():
        assert L.lib.lora_status_string(code).decode() == name


def _fwd(d, x=16, w0=32, a=48, b=64, bias=None, y=80, h=None, ws=4096, wsb=1 << 20):
    return L.lib.lora_linear_fwd(ctypes.byref(d), x, w0, a, b, bias, y, h, ws, wsb, None)


def test_fwd_validation_codes():
    ok = L.dims(128, 64, 64, 4, 16.0)
    # fake (never dereferenced) 16-byte-aligned addresses; validation fails first
    assert _fwd(L.dims(128, 60, 64, 4, 16.0)) == 2            # d_in % 8
    assert "d_in" in L.lib.lora_last_error().decode()
    assert _fwd(L.dims(128, 64, 0, 4, 16.0)) == 2             # d_out
    assert _fwd(L.dims(-1, 64, 64, 4, 16.0)) == 2             # tokens
    assert _fwd(L.dims(128, 64, 64, 0, 16.0)) == 2            # rank
    assert _fwd(L.dims(128, 64, 64, 65, 16.0)) == 4           # rank > 64
    assert _fwd(L.dims(128, 64, 64, 4, float("nan"))) == 1    # alpha
    assert L.lib.lora_linear_fwd(None, 16, 32, 48, 64, None, 80, None, 4096, 1 << 20, None) == 1
    assert _fwd(ok, x=None) == 1                              # NULL input
    assert _fwd(ok, x=24) == 3                                # misaligned
    assert "x" in L.lib.lora_last_error().decode()
    assert _fwd(ok, wsb=8) == 7                               # workspace too small
    assert _fwd(ok, ws=None) == 7
    # output overlapping an input
    assert _fwd(ok, x=1 << 20, y=(1 << 20) + 16 * 1024) == 1


def test_bwd_and_merge_validation_codes():
    d = L.dims(128, 64, 64, 4, 16.0)
    need = L.lora_linear_bwd_workspace_bytes(d)
    assert need > 0
    f = L.lib.lora_linear_bwd
    base = dict(x=1 << 30, w0=2 << 30, a=3 << 30, b=4 << 30, h=None, dy=5 << 30, dx=6 << 30,
                da=7 << 30, db=8 << 30, acc=0, ws=9 << 30, wsb=need)

    def call(**kw):
        p = dict(base, **kw)
        return f(ctypes.byref(kw.pop("d", d)), p["x"], p["w0"], p["a"], p["b"], p["h"], p["dy"],
                 p["dx"], p["da"], p["db"], p["acc"], p["ws"], p["wsb"], None)

    assert call(dy=None) == 1
    assert call(acc=2) == 1
    assert call(db=(8 << 30) + 4) == 3
    assert call(wsb=need - 1) == 7
    assert call(da=1 << 30) == 1       # dA aliases x
    m = L.lib.lora_merge
    assert m(ctypes.byref(L.dims(0, 64, 64, 4, 16.0)), 1 << 30, 2 << 30, 3 << 30, (1 << 30) + 64, None) == 1
    assert m(ctypes.byref(L.dims(0, 64, 64, 4, 16.0)), 1 << 30, 2 << 30, 3 << 30, None, None) == 1
    assert m(ctypes.byref(L.dims(0, 64, 12, 4, 16.0)), 1 << 30, 2 << 30, 3 << 30, 4 << 30, None) == 2


def test_workspace_sizes_scale_with_shape():
    f = L.lora_linear_fwd_workspace_bytes
    assert f(L.dims(2048, 4096, 4096, 8, 16.0)) >= 4096 * 8 * 2       # B8 [m, roundup(r, 8)]
    assert f(L.dims(2048, 4096, 4096, 8, 16.0)) == f(L.dims(7, 4096, 4096, 8, 16.0))
    # opt-in stream-K schedule (LORA_STREAMK=1): launches with >= 32 tiles also get one
    # fp32 128 x 256 partial accumulator slot per CTA of the 148-SM grid
    slots = 148 * 128 * 256 * 4
    base = f(L.dims(2048, 4096, 4096, 8, 16.0))
    os.environ["LORA_STREAMK"] = "1"
    try:
        assert f(L.dims(2048, 4096, 4096, 8, 16.0)) == base + slots
        assert f(L.dims(7, 4096, 4096, 8, 16.0)) == f(L.dims(7, 4096, 4096, 8, 16.0))
    finally:
        del os.environ["LORA_STREAMK"]
    b = L.lora_linear_bwd_workspace_bytes
    assert b(L.dims(4096, 4096, 11008, 16, 16.0)) > b(L.dims(2048, 4096, 11008, 16, 16.0))
    assert b(L.dims(128, 60, 64, 4, 16.0)) == 0          # invalid dims -> 0


def test_no_device_is_an_error_not_a_fallback():
    """With valid arguments and no usable B200, the call fails loudly
    (LORA_ERR_CUDA / LORA_ERR_UNSUPPORTED) instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    d = L.dims(128, 64, 64, 4, 16.0)
    st = _fwd(d, x=1 << 30, w0=2 << 30, a=3 << 30, b=4 << 30, y=5 << 30, ws=6 << 30)
    assert st in (4, 5)
    assert L.lib.lora_device_check() in (4, 5)


def test_dropout_validation_codes():
    """lora_linear_{fwd,bwd}_dropout / lora_dropout_mask reject a bad p before
    anything else (LoRA dropout; include/lora.h)."""
    d = L.dims(128, 64, 64, 4, 16.0)
    for p in (1.0, -0.5, float("nan"), float("inf")):
        dr = L.lora_dropout(p, 1, 2)
        assert L.lib.lora_linear_fwd_dropout(ctypes.byref(d), ctypes.byref(dr), 16, 32, 48, 64, None, 80, None,
                                             4096, 1 << 20, None) == 1
        assert "dropout p" in L.lib.lora_last_error().decode()
        assert L.lib.lora_linear_bwd_dropout(ctypes.byref(d), ctypes.byref(dr), 16, 32, 48, 64, None, 96, None,
                                             None, None, 0, 4096, 1 << 20, None) == 1
        assert L.lib.lora_dropout_mask(8, 8, ctypes.byref(dr), 16, None) == 1
    dr = L.lora_dropout(0.1, 1, 2)
    assert L.lib.lora_dropout_mask(8, 8, None, 16, None) == 1
    assert L.lib.lora_dropout_mask(-1, 8, ctypes.byref(dr), 16, None) == 2
    # dropout workspaces hold at least the plain ones (+ M . x and the keep bits for the backward)
    assert L.lib.lora_linear_fwd_dropout_workspace_bytes(ctypes.byref(d)) >= L.lora_linear_fwd_workspace_bytes(d)
    assert (L.lib.lora_linear_bwd_dropout_workspace_bytes(ctypes.byref(d)) >=
            L.lora_linear_bwd_workspace_bytes(d) + 128 * 64 * 2)


def test_adam_validation_codes():
    """lora_adam_step validates before any launch."""
    hp = L.lora_adam_hparams(1e-3, 0.9, 0.999, 1e-8)
    t = (L.lora_adam_tensor * 1)(L.lora_adam_tensor(16, None, 32, 48, 64, 8))
    assert L.lib.lora_adam_step(0, t, ctypes.byref(hp), 1, None) == 1            # count
    assert L.lib.lora_adam_step(65, t, ctypes.byref(hp), 1, None) == 1
    assert L.lib.lora_adam_step(1, t, None, 1, None) == 1
    assert L.lib.lora_adam_step(1, t, ctypes.byref(hp), 0, None) == 1            # step >= 1
    bad = L.lora_adam_hparams(1e-3, 1.0, 0.999, 1e-8)
    assert L.lib.lora_adam_step(1, t, ctypes.byref(bad), 1, None) == 1           # beta1 < 1
    t6 = (L.lora_adam_tensor * 1)(L.lora_adam_tensor(16, None, 32, 48, 64, 6))
    assert L.lib.lora_adam_step(1, t6, ctypes.byref(hp), 1, None) == 2           # numel % 4
    tn = (L.lora_adam_tensor * 1)(L.lora_adam_tensor(16, None, None, 48, 64, 8))
    assert L.lib.lora_adam_step(1, tn, ctypes.byref(hp), 1, None) == 1           # NULL grad
    ta = (L.lora_adam_tensor * 1)(L.lora_adam_tensor(16, 40, 32, 48, 64, 8))
    assert L.lib.lora_adam_step(1, ta, ctypes.byref(hp), 1, None) == 3           # misaligned master


def test_dropout_kept_buffers_validation():
    """lora_dropout.keep_bits / masked_x (include/lora.h): misaligned buffers are
    rejected with LORA_ERR_ALIGN before anything runs, naming the field; negative
    offsets or a column offset that is not a multiple of 8 are LORA_ERR_INVALID;
    the struct layout matches the header."""
    assert ctypes.sizeof(L.lora_dropout) == 56
    assert [f[0] for f in L.lora_dropout._fields_] == ["p", "seed", "offset", "keep_bits", "masked_x", "row_offset",
                                                       "col_offset"]
    d = L.dims(128, 64, 64, 4, 16.0)
    for kb, mx, name in ((1 << 20 | 4, None, "keep_bits"), (None, 1 << 20 | 8, "masked_x")):
        dr = L.lora_dropout(0.1, 1, 2, kb, mx)
        assert L.lib.lora_linear_fwd_dropout(ctypes.byref(d), ctypes.byref(dr), 16, 32, 48, 64, None, 80, None,
                                             4096, 1 << 20, None) == 3
        assert name in L.lib.lora_last_error().decode()
        assert L.lib.lora_linear_bwd_dropout(ctypes.byref(d), ctypes.byref(dr), 16, 32, 48, 64, None, 96, None,
                                             None, None, 0, 4096, 1 << 20, None) == 3
    for r0, c0 in ((-1, 0), (0, -8), (0, 4)):
        dr = L.lora_dropout(0.1, 1, 2, None, None, r0, c0)
        assert L.lib.lora_linear_fwd_dropout(ctypes.byref(d), ctypes.byref(dr), 16, 32, 48, 64, None, 80, None,
                                             4096, 1 << 20, None) == 1
        assert "offset" in L.lib.lora_last_error().decode()
        assert L.lib.lora_dropout_mask(8, 8, ctypes.byref(dr), 16, None) == 1

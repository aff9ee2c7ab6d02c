"""lora_write_safetensors (host tensors): the
file is the safetensors layout a Hugging Face loader reads -- checked by an
independent reader (tests/safetensors_read.py): header length, 8-byte padding,
dtype / shape / contiguous data_offsets in order, the bytes themselves."""
import numpy as np
import torch

import paper_2403_11366_b200 as L
from tests.safetensors_read import read_safetensors


def test_write_safetensors_roundtrip(tmp_path):
    g = torch.Generator().manual_seed(5)
    ts = {
        "model.layers.0.self_attn.q_proj.weight": torch.randn(24, 16, generator=g).to(torch.bfloat16),
        "model.layers.0.input_layernorm.weight": torch.randn(16, generator=g),
        "weird \"name\"\\x": torch.randn(3, 1, 2, generator=g).to(torch.bfloat16),
        "empty": torch.zeros(0, 4),
    }
    p = tmp_path / "m.safetensors"
    L.write_safetensors(p, ts)
    got, meta, hl = read_safetensors(p)
    assert hl % 8 == 0 and meta.get("format") == "pt"
    assert list(got) == list(ts)              # header order = file order
    off = 0
    raw = open(p, "rb").read()[8 + hl:]
    for name, t in ts.items():
        dt, shape, b = got[name]
        assert dt == ("BF16" if t.dtype == torch.bfloat16 else "F32")
        assert shape == tuple(t.shape)
        want = t.contiguous().view(torch.int16 if t.dtype == torch.bfloat16 else torch.int32).numpy().tobytes()
        assert b == want
        assert raw[off:off + len(want)] == want   # offsets are contiguous, in order
        off += len(want)
    assert off == len(raw)


def test_write_safetensors_errors(tmp_path):
    import pytest
    with pytest.raises(L.LoraError, match="cannot open"):
        L.write_safetensors(tmp_path / "no" / "such" / "dir.safetensors", {"a": torch.zeros(2)})
    with pytest.raises(ValueError):
        L.write_safetensors(tmp_path / "x.safetensors", {"a": torch.zeros(2, dtype=torch.int32)})

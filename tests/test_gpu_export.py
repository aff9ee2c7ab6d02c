"""lora_export_merged (Listing 4): merged
entries are W' = RNE_bf16(W0 + s B A) (Eq. 1 line 2) -- >= 99.9%
bit-equal to the rounded fp64 oracle, the rest within one bf16 ulp, exactly the
bits lora_merge returns -- and plain entries are written unchanged; the file is
read back by an independent safetensors reader."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import make_lora_inputs  # noqa: E402
from tests.gpu_util import bits_of, dev_bf16, rne_bf16_f64  # noqa: E402
from tests.safetensors_read import read_safetensors  # noqa: E402


def test_export_merged_llama_names(oracle_mod, tmp_path):
    import paper_2403_11366_b200 as L
    shapes = {"q_proj": (512, 384, 8), "v_proj": (256, 384, 16)}   # (d_out, d_in, r)
    entries, refs = [], {}
    for i, (nm, (m, n, r)) in enumerate(shapes.items()):
        d = make_lora_inputs(1, n, m, r, seed=990 + i)
        w0, a, b = dev_bf16(d["w0"]), dev_bf16(d["a"]), dev_bf16(d["b"])
        name = f"model.layers.0.self_attn.{nm}.weight"
        entries.append((name, w0, a, b, 16.0))
        refs[name] = (rne_bf16_f64(oracle_mod.lora_merge(d["w0"], d["a"], d["b"], 16.0)),
                      bits_of(L.lora_merge(w0, a, b, 16.0)))
    norm = torch.randn(384, device="cuda")
    entries.append(("model.layers.0.input_layernorm.weight", norm))
    p = tmp_path / "merged.safetensors"
    L.export_merged(p, entries)
    got, meta, _ = read_safetensors(p)
    assert meta["format"] == "pt"
    for name, (ref, merge_bits) in refs.items():
        dt, shape, raw = got[name]
        assert dt == "BF16" and shape == ref.shape
        bits = np.frombuffer(raw, dtype=np.uint16).reshape(shape)
        assert np.array_equal(bits, merge_bits)            # the same bits as lora_merge
        vals = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        assert np.mean(vals == ref) >= 0.999
        assert np.all(np.abs(vals - ref) <= np.abs(ref) * 2.0 ** -7 + 1e-30)
    dt, shape, raw = got["model.layers.0.input_layernorm.weight"]
    assert dt == "F32" and shape == (384,)
    assert np.array_equal(np.frombuffer(raw, dtype=np.float32), norm.cpu().numpy())

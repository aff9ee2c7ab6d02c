"""A plain reader of the safetensors format (test helper): u64 LE header length,
JSON header, raw bytes.  Returns ({name: (dtype, shape, raw bytes)}, metadata)."""
import json
import struct


def read_safetensors(path):
    with open(path, "rb") as f:
        blob = f.read()
    (hl,) = struct.unpack("<Q", blob[:8])
    header = json.loads(blob[8:8 + hl].decode())
    meta = header.pop("__metadata__", {})
    data = blob[8 + hl:]
    out = {}
    for name, d in header.items():
        b, e = d["data_offsets"]
        out[name] = (d["dtype"], tuple(d["shape"]), data[b:e])
    return out, meta, hl

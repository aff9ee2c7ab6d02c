"""Decoder-layer parity at head_dim 64 (the case the first layer fuzz flagged)."""
import sys

sys.path.insert(0, ".")
import tests.test_gpu_layer as t  # noqa: E402

for case in [(307, 64, 128, 1, 3), (397, 128, 80, 2, 27), (300, 256, 704, 4, 5), (200, 512, 1024, 8, 16)]:
    try:
        t.test_layer_fwd_bwd_matches_oracle(*case)
        print(case, "PASS", flush=True)
    except AssertionError as e:
        print(case, "FAIL", str(e)[:200], flush=True)

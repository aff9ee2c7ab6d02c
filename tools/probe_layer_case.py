"""Diagnose a decoder-layer parity failure: run tests/test_gpu_layer's check on variants."""
import sys

sys.path.insert(0, ".")
import tests.test_gpu_layer as t  # noqa: E402

for case in [(103, 256, 1512, 2, 1), (103, 256, 1512, 2, 8), (104, 256, 1512, 2, 1), (103, 256, 1536, 2, 1),
             (103, 256, 1512, 2, 2), (128, 256, 1512, 2, 1), (103, 256, 1512, 1, 1)]:
    try:
        t.test_layer_fwd_bwd_matches_oracle(*case)
        print(case, "PASS", flush=True)
    except AssertionError as e:
        print(case, "FAIL", str(e)[:200], flush=True)

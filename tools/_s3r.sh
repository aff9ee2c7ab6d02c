#!/bin/bash
OUT=gpurun_out/s3r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_dropout.py tests/test_gpu_tp.py -q -x > $OUT/tests.log 2>&1; tail -25 $OUT/tests.log

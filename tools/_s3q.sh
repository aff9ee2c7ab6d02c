#!/bin/bash
# compute-sanitizer over the session-3 code paths (dropout K0 / apply, K2 dropout epilogue with helper warps,
# keep_bits / masked_x), small shapes
OUT=gpurun_out/s3q; mkdir -p $OUT
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_dropout.py -q -x -k "parity or keep_bits or grouped or recompute" > $OUT/memcheck_dropout.log 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck_dropout.log
tail -4 $OUT/memcheck_dropout.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_dropout.py -q -x -k "parity and 300" > $OUT/synccheck_dropout.log 2>&1; echo "synccheck rc=$?" >> $OUT/synccheck_dropout.log
tail -4 $OUT/synccheck_dropout.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_dropout.py -q -x -k "keep_bits_grouped" > $OUT/racecheck_dropout.log 2>&1; echo "racecheck rc=$?" >> $OUT/racecheck_dropout.log
tail -6 $OUT/racecheck_dropout.log

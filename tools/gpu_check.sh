#!/bin/bash
# Iteration check on one B200: build, GPU tests, a short bench run.
set -u
OUT=gpurun_out/${1:-check}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 600 python bench.py --steps 50 --warmup 5 > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log
tail -3 $OUT/gpu_tests.log
tail -c 3000 $OUT/bench.log

#!/bin/bash
OUT=gpurun_out/s3n; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_dropout.py -q -x > $OUT/dropout_tests.log 2>&1; tail -2 $OUT/dropout_tests.log
for v in base k0nopipe base k0nopipe; do
  if [ $v = base ]; then unset LORA_LIB_PATH; else export LORA_LIB_PATH=build/probe/liblora_$v.so; fi
  timeout 300 python bench.py --dropout 0.05 --steps 30 --warmup 5 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']; print('$v', round(d['ms_per_step']*1e3,1), 'K1', round(k['K1_fwd']['us'],1), 'K2', round(k['K2_dx']['us'],1))"
done
unset LORA_LIB_PATH
timeout 300 python bench.py --config cfg3 --dropout 0.05 --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']; print('cfg3', round(d['ms_per_step']*1e3,1), 'K1', round(k['K1_fwd']['us'],1), 'K2', round(k['K2_dx']['us'],1))"

#!/bin/bash
# K2 dropout-mode epilogue: which part of the q M . (gh A) term costs the ~12 us
OUT=gpurun_out/s3p; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_dropout.py -q -x 2>&1 | tail -1
for v in base nofma nolds nohfma base; do
  if [ $v = base ]; then unset LORA_LIB_PATH; else export LORA_LIB_PATH=build/probe/liblora_$v.so; fi
  timeout 300 python bench.py --dropout 0.05 --steps 30 --warmup 5 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']; print('$v', round(d['ms_per_step']*1e3,1), 'K1', round(k['K1_fwd']['us'],1), 'K2', round(k['K2_dx']['us'],1))"
done

#!/bin/bash
# K2 dropout epilogue: rolled j loop (16x smaller code) vs unrolled
for v in base rolled base rolled; do
  if [ $v = base ]; then unset LORA_LIB_PATH; else export LORA_LIB_PATH=build/probe/liblora_$v.so; fi
  timeout 300 python bench.py --dropout 0.05 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']; print('$v', round(d['ms_per_step']*1e3,1), 'K1', round(k['K1_fwd']['us_median'],1), 'K2', round(k['K2_dx']['us_median'],1), d['parity']['pass'])"
done

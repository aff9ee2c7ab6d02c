#!/bin/bash
OUT=gpurun_out/s3h; mkdir -p $OUT
for v in base dropnofma stg0; do
  if [ $v = base ]; then unset LORA_LIB_PATH; else export LORA_LIB_PATH=build/probe/liblora_$v.so; fi
  for p in 0.05 0; do
  timeout 300 python bench.py --dropout $p --steps 30 --warmup 5 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']; print('$v p=$p', round(d['ms_per_step']*1e3,1), 'K1', round(k['K1_fwd']['us'],1), 'K2', round(k['K2_dx']['us'],1), 'K3', round(k['K3_dA_dB']['us'],1))"
  done
done

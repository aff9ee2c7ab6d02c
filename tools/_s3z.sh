#!/bin/bash
# knob sweep with the final code (PDL on): K3 token split at cfg2, merge tile width
for s in auto 2 auto 2; do
  if [ $s = auto ]; then unset LORA_K3_S; else export LORA_K3_S=$s; fi
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-parity 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['hbm_bound_kernels']['merge']; print('K3_S=$s', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'merge', round(m['us'],1))"
done
unset LORA_K3_S
for bn in 128 64 128 64; do
  LORA_MERGE_BN=$bn timeout 300 python tools/prof_merge.py 2>&1 | grep "4096x4096 r8\|28672" | sed "s/^/BN=$bn /"
done

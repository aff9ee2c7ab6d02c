#!/bin/bash
# R19 evidence: tensor-core K3 vs the warp-shuffle CUDA-core K3 (LORA_K3=cluster) at r = 8 (cfg2) and r = 16 (cfg3)
OUT=gpurun_out/s3o; mkdir -p $OUT
for c in cfg2 cfg3; do for k in mma cluster; do
  if [ $k = mma ]; then unset LORA_K3; else export LORA_K3=cluster; fi
  timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > $OUT/bench_${c}_$k.json
  python -c "import json; d=json.load(open('$OUT/bench_${c}_$k.json')); k3=d['kernels_in_step']['K3_dA_dB']; g=d.get('hbm_bound_kernels',{}).get('grads_only',{}); print('$c K3=$k', 'step', round(d['ms_per_step']*1e3,1), 'us', round(d['value'],1), 'TFLOP/s', 'K3 alone after K2', round(k3['us'],1), 'us', round(k3['gbs']), 'GB/s', 'exposed', round(k3['exposed_in_step_us'],1), '| grads_only', round(g.get('us',0),1), 'us', round(g.get('gbs',0)), 'GB/s', 'parity', d['parity']['pass'])"
done; done
unset LORA_K3

for c in cfg2 cfg3; do for S in auto 1 2 3; do
  if [ $S = auto ]; then unset LORA_K3_S; else export LORA_K3_S=$S; fi
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']['K3_dA_dB']; print('$c S=$S', round(d['value'],1), round(d['ms_per_step'],4), 'K3', round(k['us'],1), 'us', round(k['gbs']), 'GB/s')"
done; done

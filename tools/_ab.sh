timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_path.py -q -x 2>&1 | tail -2
for rep in 1 2; do for v in tma notma; do
  if [ $v = notma ]; then export LORA_LIB_PATH=$PWD/paper_2403_11366_b200/liblora_notma.so; else unset LORA_LIB_PATH; fi
  for c in cfg2 cfg3; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']; print('$v $c', round(d['value'],1), round(d['ms_per_step'],4), 'K1', round(k['K1_fwd']['us'],1), 'K2', round(k['K2_dx']['us'],1), d['clocks']['sm_mhz'])"
  done
done; done

#!/bin/bash
OUT=gpurun_out/s3l; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_dropout.py -q -x > $OUT/dropout_tests.log 2>&1; tail -3 $OUT/dropout_tests.log
for i in 1 2; do timeout 300 python bench.py --dropout 0.05 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_in_step']; print('drop', round(d['ms_per_step']*1e3,1), 'K1', round(k['K1_fwd']['us'],1), 'K2', round(k['K2_dx']['us'],1), 'K3', round(k['K3_dA_dB']['us'],1), d['parity']['pass'], d['parity']['relF_max_over_linears'])"; done
timeout 300 python bench.py --config cfg3 --dropout 0.05 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 drop', round(d['value'],1), round(d['ms_per_step']*1e3,1), d['parity']['pass'])"
timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['value'],1), round(d['ms_per_step']*1e3,1), d['parity']['pass'])"

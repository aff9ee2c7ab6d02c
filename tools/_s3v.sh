#!/bin/bash
OUT=gpurun_out/s3v; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tp.py tests/test_gpu_dropout.py -q -x > $OUT/tests.log 2>&1; tail -3 $OUT/tests.log
for c in cfg2 cfg3; do
timeout 600 python bench.py --config $c --force-tp --dropout 0.05 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c force-tp dropout grouped', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['parity'] and d['parity']['pass'])"
done
timeout 600 python bench.py --config cfg3 --force-tp --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 force-tp', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['parity'] and d['parity']['pass'])"

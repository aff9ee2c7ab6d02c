#!/bin/bash
OUT=gpurun_out/s3s; mkdir -p $OUT
for c in cfg2 cfg3; do
timeout 600 python bench.py --config $c --force-tp --dropout 0.05 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -3 > $OUT/bench_${c}_tp_drop.log
grep '^{' $OUT/bench_${c}_tp_drop.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c force-tp dropout', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['parity'] and d['parity']['pass'], d['config'].get('parallelism'))" || tail -3 $OUT/bench_${c}_tp_drop.log
done

#!/bin/bash
# session-3 iteration: dropout K0 rewrite + host-gap probe
OUT=gpurun_out/s3a; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_dropout.py -q -x > $OUT/dropout_tests.log 2>&1; tail -3 $OUT/dropout_tests.log
timeout 300 python tools/probe_gap.py > $OUT/gap.txt 2>&1; cat $OUT/gap.txt
for p in 0.05 0; do timeout 300 python bench.py --dropout $p --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_drop$p.log 2>&1; grep '^{' $OUT/bench_drop$p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p=$p', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['parity']['pass'] if d.get('parity') else None, json.dumps(d['kernels_in_step']['K1_fwd']))"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_drop.csv python bench.py --dropout 0.05 --steps 2 --warmup 1 --graph off --no-cpu-baseline --no-parity > /dev/null 2>&1
python tools/ncu_summary.py launches $OUT/launches_drop.csv $OUT/launches_drop.json > /dev/null 2>&1; python -c "import json; d=json.load(open('$OUT/launches_drop.json')); print(json.dumps(d)[:3000])"

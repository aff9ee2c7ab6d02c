OUT=gpurun_out/r02_final
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; tail -1 $OUT/gpu_tests.log
for c in cfg2 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 > $OUT/bench_$c.json.log 2>&1; grep '^{' $OUT/bench_$c.json.log > $OUT/bench_$c.json; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | grep '^{' > $OUT/bench_reference.json
LORA_COOP=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg3_force_tp.csv python bench.py --config cfg3 --force-tp --steps 1 --warmup 1 --graph off --no-cpu-baseline --no-parity > /dev/null 2>&1
LORA_COOP=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --graph off --no-cpu-baseline --no-parity > /dev/null 2>&1
for f in $OUT/bench_cfg*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],4), d['roofline']['frac'], d['roofline'].get('frac_of_sustained'), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['parity'] and d['parity']['pass'])"; done
grep -c -i nccl $OUT/launches_cfg3_force_tp.csv

#!/bin/bash
# Round-2 closing evidence (session 3) on one B200, via gpurun from the repo root.
set -u
OUT=gpurun_out/${FINAL_OUT:-r02_final2}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; tail -1 $OUT/gpu_tests.log
for i in 1 2 3; do timeout 600 python bench.py --steps 200 --warmup 10 2>/dev/null | grep '^{' >> $OUT/bench_cfg2_runs.jsonl; done
for c in cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' > $OUT/bench_$c.json; done
timeout 600 python bench.py --dropout 0.05 --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | grep '^{' > $OUT/bench_cfg2_dropout.json
timeout 600 python bench.py --dropout 0.05 --dropout-mask redraw --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | grep '^{' > $OUT/bench_cfg2_dropout_redraw.json
timeout 600 python bench.py --config cfg3 --dropout 0.05 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' > $OUT/bench_cfg3_dropout.json
timeout 600 python bench.py --layer layer7b --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' > $OUT/bench_layer7b.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | grep '^{' > $OUT/bench_reference.json
LORA_COOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --graph off --no-cpu-baseline --no-parity > /dev/null 2>&1
LORA_COOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2_dropout.csv python bench.py --dropout 0.05 --steps 2 --warmup 1 --graph off --no-cpu-baseline --no-parity > /dev/null 2>&1
LORA_COOP=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_fused_gemm -s 4 -c 2 -o $OUT/k1k2_cfg2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --graph off > $OUT/ncu_full_k1k2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dropout_h_group|merge_mma" -c 2 -o $OUT/k0_merge python bench.py --dropout 0.05 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --graph off > $OUT/ncu_full_k0.log 2>&1
for f in $OUT/bench_cfg2_runs.jsonl $OUT/bench_cfg3.json $OUT/bench_cfg4.json $OUT/bench_cfg5.json $OUT/bench_cfg2_dropout.json $OUT/bench_cfg2_dropout_redraw.json $OUT/bench_cfg3_dropout.json; do python - "$f" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    d = json.loads(line)
    r = d.get("roofline", {})
    print(sys.argv[1].split("/")[-1], round(d["value"], 1), round(d["ms_per_step"] * 1e3, 1), "us", r.get("frac"), r.get("frac_of_sustained"),
          d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("parity") and d["parity"]["pass"])
PY
done
ls -la $OUT

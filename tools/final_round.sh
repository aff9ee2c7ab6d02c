#!/bin/bash
# Round-end evidence on one B200 (run via gpurun from the repo root):
# bench lines for every config, the reference (oracle) arm, the smoke test,
# the ncu launch list of the default bench and full ncu captures of K1/K2/K3.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 120 python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1
for i in 1 2 3 4 5; do timeout 400 python bench.py | tail -1 >> $OUT/bench_cfg2_runs.jsonl; done
for c in cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline | tail -1 >> $OUT/bench_${c}_runs.jsonl; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 | tail -1 > $OUT/bench_reference.json
timeout 400 python bench.py --dropout 0.05 --no-cpu-baseline | tail -1 > $OUT/bench_cfg2_dropout.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --graph off > $OUT/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_fused_gemm -s 4 -c 2 \
    -o $OUT/k1k2_cfg2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --graph off > $OUT/ncu_full_k1k2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grad_mma -s 2 -c 1 \
    -o $OUT/k3_cfg2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --graph off > $OUT/ncu_full_k3.log 2>&1
ls -la $OUT

mkdir -p gpurun_out/tpc2
timeout 300 python -m pytest tests/test_gpu_symm.py -x -q 2>&1 | tail -2
for c in cfg2 cfg3; do for rep in 1 2; do
timeout 300 python bench.py --config $c --force-tp --comm fused --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/tpc2/$c.$rep.log 2>&1
echo "$c/$rep: $(grep -c 'never published' gpurun_out/tpc2/$c.$rep.log) unpublished; $(grep '^{"metric"' gpurun_out/tpc2/$c.$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["ms_per_step"], d["parity"]["pass"])' 2>/dev/null)"
done; done

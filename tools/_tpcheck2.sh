mkdir -p gpurun_out/tpc4
timeout 300 python -m pytest tests/test_gpu_symm.py -x -q 2>&1 | tail -2
for c in cfg2 cfg3; do for cm in nccl fused; do
timeout 300 python bench.py --config $c --force-tp --comm $cm --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/tpc4/$c.$cm.log 2>&1
echo "$c/$cm: $(grep -c 'never published' gpurun_out/tpc4/$c.$cm.log) unpublished; $(grep '^{"metric"' gpurun_out/tpc4/$c.$cm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["ms_per_step"], d["parity"]["pass"], d["config"]["tp_comm"])' 2>/dev/null)"
done; done

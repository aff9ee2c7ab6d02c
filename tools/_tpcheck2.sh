mkdir -p gpurun_out/tpc3
for c in cfg2 cfg3; do for cm in nccl fused; do
timeout 300 python bench.py --config $c --force-tp --comm $cm --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/tpc3/$c.$cm.log 2>&1
echo "$c/$cm: $(grep '^{"metric"' gpurun_out/tpc3/$c.$cm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["ms_per_step"], d["parity"]["pass"], d["gpu_launches"])' 2>/dev/null)"
done; done

mkdir -p gpurun_out/layer
LORA_COOP=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/layer/launches_layer7b.csv python bench.py --layer layer7b --steps 1 --warmup 3 --graph off > gpurun_out/layer/ncu_run.log 2>&1
tail -3 gpurun_out/layer/ncu_run.log

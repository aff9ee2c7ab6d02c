mkdir -p gpurun_out/b3
for c in cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/b3/bench_$c.json; done
for S in 1 2 3 4; do LORA_K3_S=$S timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S=$S', round(d['value'],1), d['kernels_in_step']['K3_dA_dB'])"; done
LORA_COOP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lora_fused_gemm_kernel|grad_mma_kernel" -s 8 -c 3 -o gpurun_out/b3/k123 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --graph off > gpurun_out/b3/ncu.log 2>&1
tail -2 gpurun_out/b3/ncu.log

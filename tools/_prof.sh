mkdir -p gpurun_out/r02k3
ncu --set full --clock-control none --import-source on -k regex:grad_mma_kernel -s 4 -c 1 -o gpurun_out/r02k3/k3 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --graph off > gpurun_out/r02k3/ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lora_fused_gemm_kernel -s 6 -c 2 -o gpurun_out/r02k3/k12 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --graph off > gpurun_out/r02k3/ncu_k12.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k3/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
ls -la gpurun_out/r02k3

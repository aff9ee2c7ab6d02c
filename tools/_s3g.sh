#!/bin/bash
OUT=gpurun_out/s3g; mkdir -p $OUT
LORA_COOP=0 ncu --set full --clock-control none --import-source on -k regex:lora_fused_gemm_kernel -s 3 -c 1 -o $OUT/k2drop python bench.py --dropout 0.05 --steps 1 --warmup 3 --graph off --no-cpu-baseline --no-parity > $OUT/ncu1.log 2>&1
LORA_COOP=0 ncu --set full --clock-control none --import-source on -k regex:lora_fused_gemm_kernel -s 3 -c 1 -o $OUT/k2plain python bench.py --steps 1 --warmup 3 --graph off --no-cpu-baseline --no-parity > $OUT/ncu2.log 2>&1
ls $OUT

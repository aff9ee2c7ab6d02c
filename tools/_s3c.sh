#!/bin/bash
OUT=gpurun_out/s3c; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:"dropout_(h|apply)_group" -c 2 -o $OUT/k0 python bench.py --dropout 0.05 --steps 1 --warmup 1 --graph off --no-cpu-baseline --no-parity > $OUT/ncu.log 2>&1
ls -la $OUT

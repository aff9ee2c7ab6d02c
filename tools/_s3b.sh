#!/bin/bash
OUT=gpurun_out/s3b; mkdir -p $OUT
export LORA_LIB_PATH=build/probe/liblora_k3probe.so
timeout 300 python tools/probe_k3b.py > $OUT/probe.txt 2>&1
SWEEP_S=1 LORA_K3_NOCLUSTER=1 timeout 300 python tools/probe_k3b.py > $OUT/probe_nocluster.txt 2>&1
SWEEP_S=auto LORA_K3_OVERLAP=0 timeout 300 python tools/probe_k3b.py > $OUT/probe_nooverlap.txt 2>&1
tail -n 20 $OUT/*.txt

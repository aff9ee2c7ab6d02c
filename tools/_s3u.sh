#!/bin/bash
OUT=gpurun_out/s3u; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropout.py tests/test_gpu_bench_path.py -q -x > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-parity 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['hbm_bound_kernels']['grads_only']; print('step', round(d['ms_per_step']*1e3,1), 'grads_only', round(g['us'],1), 'us', round(g['gbs']), 'GB/s', round(g['frac_of_same_bytes_copy'],3), 'of copy')"; done
timeout 300 python tools/probe_k3b.py 2>&1 | grep '"dx": false' | head -4

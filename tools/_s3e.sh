#!/bin/bash
OUT=gpurun_out/s3e; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_dropout.py -q -x > $OUT/dropout_tests.log 2>&1; tail -3 $OUT/dropout_tests.log
for dm in kept redraw; do timeout 300 python bench.py --dropout 0.05 --dropout-mask $dm --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_drop_$dm.log 2>&1; grep '^{' $OUT/bench_drop_$dm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$dm', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['parity']['pass'] if d.get('parity') else None, json.dumps(d['kernels_in_step']))"; done
LORA_COOP=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_drop.csv python bench.py --dropout 0.05 --steps 2 --warmup 1 --graph off --no-cpu-baseline --no-parity > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open('$OUT/launches_drop.csv')))
hdr=None
for r in rows[-40:]:
    if len(r)>5 and r[0]=='ID': hdr=r; continue
for r in rows:
    if len(r)>5 and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum' and 'lora' in d['Kernel Name'] and 'adam' not in d['Kernel Name']:
            print(d['Kernel Name'][:60], d['Metric Value'])
PY
LORA_COOP=0 ncu --set full --clock-control none --import-source on -k regex:"lora_fused_gemm_kernel<2|dropout_h_group" -c 2 -o $OUT/k2drop python bench.py --dropout 0.05 --steps 1 --warmup 1 --graph off --no-cpu-baseline --no-parity > $OUT/ncu1.log 2>&1
LORA_COOP=0 ncu --set full --clock-control none --import-source on -k regex:"lora_fused_gemm_kernel<1" -c 1 -o $OUT/k2plain python bench.py --steps 1 --warmup 1 --graph off --no-cpu-baseline --no-parity > $OUT/ncu2.log 2>&1
ls $OUT

#!/bin/bash
for cfg in "SS_STATIC_PCT=100" "SS_STATIC_PCT=70 SS_CHUNK_DIV=2" "SS_STATIC_PCT=50 SS_CHUNK_DIV=2" "SS_STATIC_PCT=50 SS_CHUNK_DIV=4"; do
  env $cfg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/chunk.csv python tools/prof_step.py --layers 2 --steps 2 > /dev/null 2>&1
  python - "$cfg" << 'PY'
import csv, sys
rows = list(csv.reader(open('gpurun_out/chunk.csv'))); hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
print('cfg', sys.argv[1], [(x['Kernel Name'][12:24], x['Metric Value']) for x in data[-5:]])
PY
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg', '$cfg', 'step us', round(d['value'],1))"
done

#!/bin/bash
for v in libswiftspec.so libswiftspec_s2.so libswiftspec_s2w16.so libswiftspec_s4.so; do
  SWIFTSPEC_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/exp_$v.csv python tools/prof_step.py --layers 2 --steps 2 > /dev/null 2>&1
  python - "$v" << 'PY'
import csv, sys
v = sys.argv[1]
rows = list(csv.reader(open(f'gpurun_out/exp_{v}.csv'))); hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
print(v, [(d['Kernel Name'][12:24], d['Metric Value']) for d in data[-10:] if d['Metric Name'].startswith('gpu__time')], [d['Metric Value'] for d in data[-10:] if d['Metric Name'].startswith('launch')][:2])
PY
  SWIFTSPEC_LIB=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'step us', round(d['value'],1))"
done

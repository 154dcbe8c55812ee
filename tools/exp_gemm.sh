#!/bin/bash
for v in libswiftspec.so libswiftspec_l2w.so libswiftspec_l2wnodeq.so libswiftspec_l2wnocomp.so; do
  SWIFTSPEC_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.per_cycle_active,smsp__inst_executed.sum --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/exp_$v.csv python tools/prof_step.py --layers 2 --steps 2 > /dev/null 2>&1
  python - "$v" << 'PY'
import csv, sys
v = sys.argv[1]
rows = list(csv.reader(open(f'gpurun_out/exp_{v}.csv'))); hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
for d in data[-15:]:
    print(v, d['Kernel Name'][12:24], d['Metric Name'][:28], d['Metric Value'])
PY
done

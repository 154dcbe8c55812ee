#!/bin/bash
# tests + bench + launch list (no full ncu capture)
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/tests.log 2>&1
tail -3 gpurun_out/tests.log
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('step us', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['step_roofline_frac'],3), 'gu frac', round(d.get('roofline',{}).get('frac',0),3))
print({k: round(v['total']/max(v['launches'],1),1) for k,v in d.get('kernel_times_us',{}).items()})
" ; tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python tools/prof_step.py --layers 4 --steps 3 > gpurun_out/launches.out 2>&1
python - << 'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches.csv'))); hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
for d in data[-11:]: print('  ', d['Kernel Name'][:40], d['Grid Size'], d['Metric Value'])
PY

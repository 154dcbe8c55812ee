#!/bin/bash
# attention variant (cluster DSMEM merge vs global merge) on the TP-rank emulation, after the row split
mkdir -p gpurun_out
for rep in 1 2; do
for kv in "" "SS_ATTN_CLUSTER=0" "SS_ATTN_CLUSTER=1"; do
  env $kv timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cl.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/cl.json')); t=d['tp_emulated']; print('$kv'.ljust(18), round(d['value'],1), {k: (round(v['us'],1), v['status_ok']) for k,v in t.items() if isinstance(v, dict)})"
done
done

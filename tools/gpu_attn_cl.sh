#!/bin/bash
# attention variant sweep at TP1 (timing): global merge vs 16-CTA cluster with smem padding
mkdir -p gpurun_out
for cfg in "0 0" "1 0" "1 120" "1 160"; do
  set -- $cfg
  SS_ATTN_CLUSTER=$1 SS_ATTN_CL_SMEM_KB=$2 timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-tp-emulate > gpurun_out/acl.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/acl.json')); print('cluster=$1 pad=$2', round(d['value'],1))"
done

#!/bin/bash
# A/B of the default grid sizing against SS_GEMM_MINU=1 (the previous default), alternating
mkdir -p gpurun_out
for rep in 1 2; do
for kv in "" "SS_GEMM_MINU=1"; do
  for c in "llama3-1b 8 1024" "llama3-8b 8 4096"; do
    set -- $c
    env $kv timeout 200 python bench.py --config $1 --T $2 --L $3 --steps 20 --warmup 5 --no-cpu-baseline --no-tp-emulate > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print('$kv'.ljust(16) or 'default', '$1 T$2', round(d['value'],1), 'ok', d['status_ok'])"
  done
  env $kv timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); t=d['tp_emulated']; print('$kv'.ljust(16), '70b T8', round(d['value'],1), {k: round(v['us'],1) for k,v in t.items() if isinstance(v, dict)})"
done
done

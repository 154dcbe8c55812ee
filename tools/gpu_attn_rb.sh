#!/bin/bash
# attention row blocks per CTA (SS_ATTN_RB cap -> more row chunks) on TP1 and the TP-rank emulation
mkdir -p gpurun_out
for rep in 1 2; do
for kv in "" "SS_ATTN_RB=2" "SS_ATTN_RB=1"; do
  env $kv timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rb.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/rb.json')); t=d['tp_emulated']; print('$kv'.ljust(14), '70b T8', round(d['value'],1), 'attn eager', round(d['kernel_times_us']['attention']['total']/80,1), {k: (round(v['us'],1), v['status_ok']) for k,v in t.items() if isinstance(v, dict)})"
done
done

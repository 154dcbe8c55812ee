#!/bin/bash
# graph-mode cost of each launch kind: bench with SS_EXP_SKIP masks (timing only)
mkdir -p gpurun_out
for m in 0 1 2 4 8 16; do
  SS_EXP_SKIP=$m timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-tp-emulate > gpurun_out/skip_$m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/skip_$m.json')); print('skip', $m, 'step us', round(d['value'],1))"
done

#!/bin/bash
# bench the product library and experiment variants incl. the TP-rank emulation (VARIANTS="a b")
mkdir -p gpurun_out
for rep in 1 2; do
for v in "" ${VARIANTS}; do
  lib=libswiftspec${v:+_$v}.so
  SWIFTSPEC_LIB=$lib timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  python - "$v" <<'PY'
import json, sys
d = json.load(open(f'gpurun_out/bench_{sys.argv[1]}.json'))
tp = {k: round(v['us'], 1) for k, v in d.get('tp_emulated', {}).items() if isinstance(v, dict)}
print(sys.argv[1] or 'product', 'step us', round(d['value'], 1), 'tp', tp, flush=True)
PY
done
done

#!/bin/bash
# bench the product library and experiment variants (VARIANTS="pf4 pf16")
mkdir -p gpurun_out
for v in "" ${VARIANTS}; do
  lib=libswiftspec${v:+_$v}.so
  SWIFTSPEC_LIB=$lib timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-tp-emulate > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  python - "$v" <<'PY'
import json, sys
d = json.load(open(f'gpurun_out/bench_{sys.argv[1]}.json'))
kt = {k: round(v['total'] / max(v['launches'], 1), 1) for k, v in d.get('kernel_times_us', {}).items()}
print(sys.argv[1] or 'product', 'step us', round(d['value'], 1), 'frac', round(d['step_roofline_frac'], 3), kt)
PY
done

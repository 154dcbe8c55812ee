#!/bin/bash
# bench T in $TS for the product library and $VARIANTS
mkdir -p gpurun_out
for v in "" ${VARIANTS}; do
  for T in ${TS:-16}; do
    lib=libswiftspec${v:+_$v}.so
    SWIFTSPEC_LIB=$lib timeout 150 python bench.py --T $T --steps 10 --warmup 3 --no-cpu-baseline --no-tp-emulate > gpurun_out/bt_${v}_$T.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/bt_${v}_$T.json')); print('${v:-product}', 'T=$T', round(d['value'],1), {k: round(v['total']/max(v['launches'],1),1) for k,v in d['kernel_times_us'].items() if k in ('qkv','gate_up_swiglu','down','o_proj')})"
  done
done

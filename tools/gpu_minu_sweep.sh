#!/bin/bash
# Grid-sizing knobs (SS_GEMM_MINU = min stream-K units per CTA, SS_GEMM_OCC = CTA/SM cap)
# on the configurations dominated by per-kernel fixed costs: 1B T=16 (TP 1) and the
# TP 8-rank emulation of the 70B step, plus the 70B TP 1 headline.
mkdir -p gpurun_out
for kv in "" "SS_GEMM_MINU=2" "SS_GEMM_MINU=4" "SS_GEMM_MINU=8" "SS_GEMM_OCC=2" "SS_GEMM_OCC=1" "SS_GEMM_OCC=2 SS_GEMM_MINU=4"; do
  env $kv timeout 200 python bench.py --config llama3-1b --T 16 --L 1024 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/sw1.json 2>/dev/null
  env $kv timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sw70.json 2>/dev/null
  python - "$kv" <<'PY'
import json, sys
a = json.load(open('gpurun_out/sw1.json')); b = json.load(open('gpurun_out/sw70.json'))
print(f"{sys.argv[1] or 'default':28s} 1B-T16 {a['value']:8.1f} us  70B-TP1 {b['value']:8.1f} us  TP8-rank {b['tp_emulated']['tp8']['us']:7.1f} TP4 {b['tp_emulated']['tp4']['us']:7.1f} TP2 {b['tp_emulated']['tp2']['us']:7.1f}", flush=True)
PY
done

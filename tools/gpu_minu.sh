#!/bin/bash
# TP8-rank emulation and TP1 step vs SS_GEMM_MINU (timing)
for m in 1 2 4 8; do
  r8=$(SKIP0_ONLY=1 SS_GEMM_MINU=$m timeout 200 python tools/tp_emul_skip.py 8 2>/dev/null | head -1 | awk '{print $5}')
  [ -n "$NO_TP1" ] || SS_GEMM_MINU=$m timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-tp-emulate > gpurun_out/minu.json 2>/dev/null
  r1=$(python -c "import json; print(round(json.load(open('gpurun_out/minu.json'))['value'],1))")
  echo "minu=$m tp8-rank ${r8} us  tp1 ${r1} us"
done

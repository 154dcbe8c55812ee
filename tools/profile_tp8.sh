#!/bin/bash
# ncu of one TP 8 rank (loopback emulation): launch list of a 2-layer step + --set full of
# the four W4 GEMM launches and the attention launch of layer 1
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tp8_launches.csv \
  python tools/prof_step.py --layers 2 --steps 3 --tp 8 > gpurun_out/tp8_launches.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|attn_kernel" -s 12 -c 5 \
  -o gpurun_out/tp8_full -f python tools/prof_step.py --layers 2 --steps 3 --tp 8 > gpurun_out/tp8_full.out 2>&1
ls -la gpurun_out/tp8_*

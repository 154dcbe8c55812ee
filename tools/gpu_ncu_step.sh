#!/bin/bash
# ncu --set full of the persistent step kernel (4 layers of 70B, one TP rank)
mkdir -p gpurun_out
TP=${TP:-8}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 2 -c 1 \
  -o gpurun_out/step_tp${TP} -f python tools/prof_step.py --layers 4 --steps 3 --tp $TP > gpurun_out/ncu_step.out 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_step.out; ls -la gpurun_out/*.ncu-rep

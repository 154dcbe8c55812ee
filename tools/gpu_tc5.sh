#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/step_check.py > gpurun_out/step_check.log 2>&1; echo "step_check rc=$?"; grep step gpurun_out/step_check.log | grep -v phase | tail -8
for tp in 1 8; do
timeout 200 python tools/step_trace.py --T 8 --tp $tp --show 1 > gpurun_out/trace_att_tp$tp.log 2>&1; echo "rc=$?"; grep -A1 "CTA 0 attention" gpurun_out/trace_att_tp$tp.log; grep "mean critical\|kernel span" gpurun_out/trace_att_tp$tp.log
done

#!/bin/bash
timeout 300 python tools/step_check.py > gpurun_out/step_check.log 2>&1; echo "step_check rc=$?"; grep step gpurun_out/step_check.log | grep -v phase | tail -8
for tp in 8 1; do
timeout 200 python tools/step_trace.py --T 8 --tp $tp --show 1 > gpurun_out/trace_tail_tp$tp.log 2>&1; echo "tp$tp rc=$?"; grep "tail of\|mean crit\|kernel span" gpurun_out/trace_tail_tp$tp.log
done

#!/bin/bash
for tp in 8 1; do
timeout 200 python tools/step_trace.py --T 8 --tp $tp --show 1 > gpurun_out/trace_tail_tp$tp.log 2>&1; echo "tp$tp rc=$?"; grep "tail of" gpurun_out/trace_tail_tp$tp.log
done

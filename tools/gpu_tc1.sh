#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/step_check.py > gpurun_out/step_check.log 2>&1; echo "step_check rc=$?"; tail -22 gpurun_out/step_check.log
timeout 300 python tools/step_trace.py --T 8 --show 1 > gpurun_out/trace_tp1_T8.log 2>&1; echo "trace rc=$?"; head -12 gpurun_out/trace_tp1_T8.log; tail -1 gpurun_out/trace_tp1_T8.log
timeout 300 python tools/step_trace.py --T 8 --tp 8 --show 1 > gpurun_out/trace_tp8_T8.log 2>&1; echo "trace rc=$?"; head -1 gpurun_out/trace_tp8_T8.log; tail -1 gpurun_out/trace_tp8_T8.log

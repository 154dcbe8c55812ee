#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/step_trace.py --T 8 --tp 1 --show 1 > gpurun_out/trace_units.log 2>&1; echo "rc=$?"; tail -20 gpurun_out/trace_units.log

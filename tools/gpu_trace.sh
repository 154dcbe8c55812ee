#!/bin/bash
# step-kernel timelines (70B TP1 and one TP8 rank) + full-size parity
mkdir -p gpurun_out
timeout 300 python tools/step_trace.py --T 8 --json gpurun_out/trace_tp1_T8.json > gpurun_out/trace_tp1.log 2>&1; echo "trace tp1 rc=$?"; cat gpurun_out/trace_tp1.log | head -40
timeout 300 python tools/step_trace.py --T 8 --tp 8 --json gpurun_out/trace_tp8_T8.json > gpurun_out/trace_tp8.log 2>&1; echo "trace tp8 rc=$?"; cat gpurun_out/trace_tp8.log | head -40
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_full.log

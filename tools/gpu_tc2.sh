#!/bin/bash
mkdir -p gpurun_out
for tp in 1 8; do for T in 8 16 32; do
timeout 200 python tools/step_trace.py --T $T --tp $tp --show 1 --json gpurun_out/trace_tp${tp}_T${T}.json > gpurun_out/trace_tp${tp}_T${T}.log 2>&1; echo "trace tp$tp T$T rc=$?"; head -1 gpurun_out/trace_tp${tp}_T${T}.log; tail -1 gpurun_out/trace_tp${tp}_T${T}.log
done; done
timeout 600 python -m pytest tests/test_tp_fakepeer.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_tp.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_tp.log

#!/bin/bash
# step-kernel timelines at TP1 / one TP8 rank, T=8 and 16
mkdir -p gpurun_out
for tp in 1 8; do for T in 8 16; do
timeout 300 python tools/step_trace.py --T $T --tp $tp --show 1 --json gpurun_out/trace_tp${tp}_T${T}.json > gpurun_out/trace_tp${tp}_T${T}.log 2>&1; echo "trace tp$tp T$T rc=$?"; head -1 gpurun_out/trace_tp${tp}_T${T}.log; tail -1 gpurun_out/trace_tp${tp}_T${T}.log
done; done
sed -n 1,12p gpurun_out/trace_tp1_T8.log
sed -n 1,12p gpurun_out/trace_tp8_T8.log

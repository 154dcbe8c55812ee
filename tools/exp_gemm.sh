#!/bin/bash
# GEMM experiment variants: serialized per-launch durations under ncu
for v in libswiftspec.so libswiftspec_nozero.so libswiftspec_nodeq.so; do
  SWIFTSPEC_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/exp_$v.csv python tools/prof_step.py --layers 2 --steps 2 > /dev/null 2>&1
done

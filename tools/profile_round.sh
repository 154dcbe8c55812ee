#!/bin/bash
# Profiling evidence for profiles/: (1) per-launch device times of the bench
# command (cold-cache, serialised), (2) ncu --set full of the dominant kernels.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"gemm_kernel|attn_kernel|prep_norm|embed_meta|commit_kernel" --csv --log-file gpurun_out/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tp-emulate > gpurun_out/bench_under_ncu.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 5 \
  -o gpurun_out/full_gemm -f python tools/prof_step.py --layers 2 --steps 2 > gpurun_out/full_gemm.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 2 -c 1 \
  -o gpurun_out/full_attn -f python tools/prof_step.py --layers 2 --steps 2 > gpurun_out/full_attn.out 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/bench_launches.csv

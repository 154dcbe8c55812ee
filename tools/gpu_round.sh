#!/bin/bash
# One gpurun session: tests, smoke, bench, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/tests.log 2>&1
tail -5 gpurun_out/tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python tools/prof_step.py --layers 4 --steps 3 > gpurun_out/launches.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 8 -c 5 \
   -o gpurun_out/prof_gemm -f python tools/prof_step.py --layers 4 --steps 2 > gpurun_out/prof_gemm.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 4 -c 1 \
   -o gpurun_out/prof_attn -f python tools/prof_step.py --layers 4 --steps 2 > gpurun_out/prof_attn.out 2>&1
ls -la gpurun_out

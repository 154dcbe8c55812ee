#!/bin/bash
# Round-2 profiling evidence (profiles/): (1) ncu launch list of the bench
# command (cold-cache, serialised), (2) DRAM traffic of the full 80-layer step
# kernel (70B TP1 T=8 and one TP8 rank), (3) ncu --set full of a 4-layer step
# kernel at TP1 and TP8 (source-level stalls).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tp-emulate > gpurun_out/r02_bench_under_ncu.out 2>&1
echo "launch list rc=$?"
for TP in 1 8; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:step_kernel -s 3 -c 1 --csv --log-file gpurun_out/r02_traffic_tp$TP.csv \
  python tools/prof_step.py --layers 80 --steps 5 --T 8 --tp $TP > gpurun_out/r02_traffic_tp$TP.out 2>&1
echo "traffic tp$TP rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 2 -c 1 \
  -o gpurun_out/r02_full_tp$TP -f python tools/prof_step.py --layers 4 --steps 3 --T 8 --tp $TP > gpurun_out/r02_full_tp$TP.out 2>&1
echo "full tp$TP rc=$?"
done
ls -la gpurun_out/r02_*

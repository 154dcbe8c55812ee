#!/bin/bash
timeout 600 compute-sanitizer --tool racecheck --print-limit 40 python tools/sanitize_step.py > gpurun_out/race.log 2>&1; echo "rc=$?"
grep -B1 -A2 "Race reported" gpurun_out/race.log | grep -v "and Read access" | head -60
tail -3 gpurun_out/race.log

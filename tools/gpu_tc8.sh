#!/bin/bash
bash tools/gpu_race.sh 2>&1 | tail -2
bash tools/gpu_tc7.sh 2>&1 | grep -v "tail of"

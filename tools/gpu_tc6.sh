#!/bin/bash
timeout 200 python tools/step_trace.py --T 8 --tp 8 --show 1 > gpurun_out/trace_att_tp8.log 2>&1; echo "rc=$?"; grep -A2 "CTA 0 attention" gpurun_out/trace_att_tp8.log

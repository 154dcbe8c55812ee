#!/bin/bash
# smoke + the GPU test suite (optionally a subset: TESTS="tests/test_x.py ...")
mkdir -p gpurun_out
timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -x --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log

#!/bin/bash
# quick correctness pass: smoke + GPU parity tests (bounded)
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/tests.log

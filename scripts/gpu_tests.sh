#!/bin/bash
# GPU parity tests with a per-test timeout (a hung kernel must not hang the box)
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -s --timeout 300 "$@" > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -40 gpurun_out/gpu_tests.log

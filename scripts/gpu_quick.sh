#!/bin/bash
# build, debug paths, GPU tests, tier sweep (decode GEMM GB/s by tier)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tests/debug_paths.py > gpurun_out/debug_paths.log 2>&1; echo "debug rc=$?"; tail -11 gpurun_out/debug_paths.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
bash scripts/tier_sweep_nobuild.sh

#!/bin/bash
# build, fast parity subset + debug paths + bench (decode + prefill legs)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python tests/debug_paths.py > gpurun_out/debug_paths.log 2>&1; echo "debug rc=$?"; cat gpurun_out/debug_paths.log | tail -12
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err

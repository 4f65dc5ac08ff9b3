#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
start=$(date +%s)
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$? in $(( $(date +%s) - start )) s"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err

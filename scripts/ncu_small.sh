#!/bin/bash
# ncu full capture of the small per-layer kernels (router, route1, combine, fold) of the decode step
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:'k_router|k_route1|k_combine|k_fold|k_gather' -s 40 -c 5 -o gpurun_out/prof_small -f python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_small.log 2>&1
tail -2 gpurun_out/ncu_small.log

#!/bin/bash
mkdir -p gpurun_out
df -h /dev/shm | tail -1; free -g | head -2
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
export DX_WATCHDOG_S=120
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_route1|k_router|k_combine|k_gather|k_fold' -s 800 -c 5 -o gpurun_out/prof_route -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep > gpurun_out/ncu_route.log 2>&1
tail -1 gpurun_out/ncu_route.log

#!/bin/bash
# ncu --set full captures: all-int4 decode GEMMs, mixed decode GEMMs, prefill GEMMs (8-layer stack)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
export DX_WATCHDOG_S=120
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 580 -c 2 -o gpurun_out/prof_int4 -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 --budget-gb 16 > gpurun_out/ncu_int4.log 2>&1
tail -2 gpurun_out/ncu_int4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 580 -c 2 -o gpurun_out/prof_mixed -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_mixed.log 2>&1
tail -2 gpurun_out/ncu_mixed.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 624 -c 2 -o gpurun_out/prof_prefill -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 > gpurun_out/ncu_prefill.log 2>&1
tail -2 gpurun_out/ncu_prefill.log

#!/bin/bash
# final ncu --set full captures: one steady-state decode gate/up + down launch of the default 48-layer bench,
# and one prefill layer (both phases) of an 8-layer stack
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
export DX_WATCHDOG_S=120
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 3560 -c 2 -o gpurun_out/prof_final_decode -f python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b > gpurun_out/ncu_fd.log 2>&1
tail -1 gpurun_out/ncu_fd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 624 -c 2 -o gpurun_out/prof_final_prefill -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 --no-batch-sweep --no-q80b > gpurun_out/ncu_fp.log 2>&1
tail -1 gpurun_out/ncu_fp.log

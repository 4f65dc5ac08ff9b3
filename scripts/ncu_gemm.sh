#!/bin/bash
# ncu --set full of the tcgen05 GEMM phases in STEADY STATE (after the controller warm-up / finalize):
# 8-layer decode stack, launches of the timed steps; then the 4k prefill leg.
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 530 -c 4 -o gpurun_out/prof_gemm_ss -f python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 280 -c 2 -o gpurun_out/prof_gemm_prefill -f python bench.py --layers 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 1 > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_full2.log

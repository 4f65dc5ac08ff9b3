#!/bin/bash
# ncu full capture of the decode GEMM with every expert at int4 (DX_GEMM_DBG=$1 selects an experiment)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for dbg in ${@:-0}; do
DX_GEMM_DBG=$dbg timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 530 -c 2 -o gpurun_out/prof_int4_d$dbg -f python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --budget-gb 16 > gpurun_out/ncu_int4_d$dbg.log 2>&1
tail -2 gpurun_out/ncu_int4_d$dbg.log
done

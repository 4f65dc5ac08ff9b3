#!/bin/bash
# ncu --set full of the decode GEMM phases in the default (mixed-tier) bench configuration; writes the
# per-launch DRAM traffic of the gate/up kernel to profiles/ffn_traffic.json and a summary to profiles/
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 200 -c 4 -o gpurun_out/prof_gemm_mixed -f python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_traffic.log 2>&1
tail -2 gpurun_out/ncu_traffic.log

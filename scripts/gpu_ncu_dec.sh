#!/bin/bash
# ncu --set full of k_dec (both phases) on the all-int4 C2 stack (budget 16 GB): bash scripts/gpu_ncu_dec.sh tag [budget]
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_dec' -s 530 -c 2 -o gpurun_out/$1 -f python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --budget-gb ${2:-16} --no-batch-sweep --no-q80b > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log

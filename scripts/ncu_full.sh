#!/bin/bash
# one ncu --set full capture of the two tcgen05 expert GEMM phases on a short C2 run
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "c1_replay or paper_shapes" > gpurun_out/gpu_tests_quick.log 2>&1
tail -2 gpurun_out/gpu_tests_quick.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 200 -c 4 -o gpurun_out/prof_gemm -f python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json

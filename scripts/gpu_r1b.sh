#!/bin/bash
# one GPU call: build, gpu tests, bench, launch list, ncu --set full of the decode GEMM phases
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -4 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 20000 -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_ll.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; cat gpurun_out/launch_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 200 -c 2 -o gpurun_out/prof_gemm -f python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log

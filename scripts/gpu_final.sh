#!/bin/bash
# round deliverables: default bench line, launch list of the timed decode step, ncu --set full of one
# steady-state gate/up + down launch of the default 48-layer bench (for the roofline traffic field)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 20000 -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_ll.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; cat gpurun_out/launch_summary.txt
export DX_WATCHDOG_S=120
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 3560 -c 2 -o gpurun_out/prof_bench_gemm -f python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log

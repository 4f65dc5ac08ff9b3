#!/bin/bash
# per-kernel launch list of the decode step (ncu, serialised, cold-ish caches) -> gpurun_out/launches.csv
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(router|route|place|gemm|combine|fold|plan|xfer|gather)' -s 300 -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 ${@} > gpurun_out/ncu_ll.log 2>&1
tail -2 gpurun_out/ncu_ll.log
python scripts/launch_summary.py gpurun_out/launches.csv

#!/bin/bash
# prefill launch list (ncu gpu__time_duration per launch), 4-layer C3 stack: bash scripts/pll.sh TAG [env...]
mkdir -p gpurun_out
TAG=$1; shift
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
K='regex:k_(router|route|place|gemm|wide|combine|fold|plan|xfer|gather|dec|scan|corr|shared)'
env "$@" timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s ${SKIP:-300} -c 200 --csv --log-file gpurun_out/${TAG}_pl.csv \
  python bench.py --batch 4096 --layers 4 --steps 2 --warmup ${WU:-1} ${BX} --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > gpurun_out/${TAG}_pll.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_pl.csv

#!/bin/bash
# One GPU round trip: build, the -m gpu tests (selection via $1, default all), a short default bench and the
# decode launch list.  Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [pytest -k expr] [tag]
set -o pipefail
mkdir -p gpurun_out
TAG=${2:-run}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$1" ] && [ "$1" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -s -k "$1" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
elif [ -z "$1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
fi
tail -3 gpurun_out/${TAG}_tests.log 2>/dev/null
timeout 600 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
if [ -z "$NO_LL" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(router|route|place|gemm|combine|fold|plan|xfer|gather|dec)' -s 300 -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b > gpurun_out/${TAG}_ncu_ll.log 2>&1
  python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv | tee gpurun_out/${TAG}_launch_summary.txt
fi

#!/bin/bash
# Round evidence at HEAD (bash scripts/gpu_evidence.sh TAG): -m gpu tests, smoke, the default bench line, the C5 line,
# the reference arm, decode and prefill launch lists, ncu --set full of the decode and prefill expert GEMMs (the decode
# capture paired launch by launch with each forward's algorithmic bytes, DX_LOG_BYTES).
set -o pipefail
T=${1:-r02}
O=gpurun_out
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/${T}_smoke.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --switch-stress > $O/${T}_c5.json 2> $O/${T}_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/${T}_bench_reference.json 2> $O/${T}_ref.err; echo "ref rc=$?"
K='regex:k_(router|route|place|gemm|wide|combine|fold|plan|xfer|gather|dec|scan|corr|shared)'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 400 -c 400 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > $O/${T}_ll.log 2>&1
python scripts/launch_summary.py $O/${T}_launches.csv > $O/${T}_launch_summary.txt; cat $O/${T}_launch_summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 300 -c 200 --csv --log-file $O/${T}_prefill_launches.csv \
  python bench.py --batch 4096 --layers 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > $O/${T}_pll.log 2>&1
python scripts/launch_summary.py $O/${T}_prefill_launches.csv > $O/${T}_prefill_launch_summary.txt; cat $O/${T}_prefill_launch_summary.txt
DX_LOG_BYTES=1 DX_WATCHDOG_S=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 200 -c 4 -o $O/${T}_ncu_decode -f \
  python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > $O/${T}_ncu_decode.log 2>&1
echo "ncu decode rc=$?"
DX_WATCHDOG_S=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_(gemm|wide)' -s 200 -c 4 -o $O/${T}_ncu_prefill -f \
  python bench.py --batch 4096 --layers 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > $O/${T}_ncu_prefill.log 2>&1
echo "ncu prefill rc=$?"

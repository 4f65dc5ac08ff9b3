#!/bin/bash
# ncu --set full of the expert GEMMs in steady state (after the warm-up finalize), decode (C2 mix, 8 layers) and
# prefill (T = 4096, 4 layers); the decode capture paired launch by launch with DX_LOG_BYTES.  bash scripts/gpu_ncu_steady.sh TAG
T=${1:-r02b}
O=gpurun_out
python __graft_entry__.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
DX_LOG_BYTES=1 DX_WATCHDOG_S=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 532 -c 4 -o $O/${T}_ncu_decode -f \
  python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > $O/${T}_ncu_decode.log 2>&1
echo "ncu decode rc=$?"
DX_WATCHDOG_S=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 272 -c 2 -o $O/${T}_ncu_prefill -f \
  python bench.py --batch 4096 --layers 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > $O/${T}_ncu_prefill.log 2>&1
echo "ncu prefill rc=$?"

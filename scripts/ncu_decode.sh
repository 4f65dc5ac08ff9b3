#!/bin/bash
# ncu --set full of the fused decode FFN kernel (4 launches of an 8-layer C2 stack), each launch paired with its
# forward's algorithmic weight bytes (DX_LOG_BYTES): bash scripts/ncu_decode.sh TAG
T=${1:-dec}; O=gpurun_out; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1 || exit 1
DX_LOG_BYTES=1 DX_WATCHDOG_S=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s ${SKIP:-296} -c 4 -o $O/${T}_ncu_decode -f \
  python bench.py --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b --no-teleport --no-prefetch-leg > $O/${T}_ncu_decode.log 2>&1
echo "ncu rc=$?"

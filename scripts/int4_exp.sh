#!/bin/bash
# decode int path experiments: DX_GEMM_DBG=0 (normal) / 3 (no scale loads), all-int4
for dbg in 4 5 6; do
  echo "== DX_GEMM_DBG=$dbg all-int4"
  DX_GEMM_DBG=$dbg timeout 300 python bench.py --steps 6 --warmup 2 --no-cpu-baseline --no-e2e --prefill-tokens 0 --budget-gb 16 --layers 16 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; x=d['extra']
print('ms/step %.2f gateup %.0f GB/s both %.0f GB/s' % (d['ms_per_step'], r['achieved'], r['ffn_both_phases_gbs']))"
done

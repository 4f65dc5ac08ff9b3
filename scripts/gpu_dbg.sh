#!/bin/bash
# all-int4 / mixed decode GEMM bandwidth under the timing-only DX_GEMM_DBG switches (4: skip the TS MMAs,
# 5: skip the dequant, 6: both), then one ncu --set full capture of the prefill GEMMs
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for b in 16 24; do for d in 0 4 5 6; do
  echo "== budget $b dbg $d"
  DX_GEMM_DBG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 --budget-gb $b > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']
print('value %.0f gateup %.0f GB/s both %.0f GB/s' % (d['value'], r['achieved'], r['ffn_both_phases_gbs']))" || tail -3 gpurun_out/sweep.err
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 624 -c 2 -o gpurun_out/prof_gemm_prefill -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 > gpurun_out/ncu_prefill.log 2>&1
tail -2 gpurun_out/ncu_prefill.log

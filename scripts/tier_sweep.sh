#!/bin/bash
# Per-tier decode GEMM bandwidth (C2 stack, B=64): mixed (24 GB), all-bf16 (60 GB), all-int4 (16 GB), each with
# the decode kernel (k_dec) and, with OLD=1, the round-1 decode configuration of k_gemm; then the timing-only
# switches of k_dec (DBG 5: no dequant, 6: no dequant and no MMA) on all-int4.
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
run() {
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b "$@" 2>/tmp/ts.err | python -c "
import json,sys
t=sys.stdin.read()
try:
  d=json.loads(t); r=d['roofline']; x=d['extra']
  print('value %.0f ms/step %.3f gateup %.0f GB/s (%.3f) both %.0f GB/s (%.3f) bytes/layer %.1f MB ffn_share %.2f route_share %.2f host %.2f' % (d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['ffn_both_phases_gbs'], r['ffn_both_frac'], x['weight_bytes_per_layer']/1e6, x['ffn_ms_share'], x['route_ms_share'], x['host_issue_ms_per_step']))
except Exception as e:
  print('FAILED', e, t[-300:])
"; tail -2 /tmp/ts.err
}
for cfg in "--budget-gb 24" "--budget-gb 60" "--budget-gb 16"; do
  echo "== k_dec $cfg"; run $cfg
  if [ -n "$OLD" ]; then echo "== old $cfg"; DX_DEC_OLD=1 run $cfg; fi
done
for dbg in 5 6; do echo "== k_dec DX_GEMM_DBG=$dbg all-int4"; DX_GEMM_DBG=$dbg run --budget-gb 16 --layers 16; done

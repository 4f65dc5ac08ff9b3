#!/bin/bash
# per-tier decode GEMM bandwidth: mixed (24 GB), all-bf16 (60 GB), all-int4 (16 GB); and the mma.sync path
for cfg in "--budget-gb 24" "--budget-gb 60" "--budget-gb 16" "--budget-gb 24 --ffn-path 1"; do
  echo "== $cfg"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 $cfg > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']
print('value %.0f ms/step %.2f gateup %.0f GB/s both %.0f GB/s bytes/layer %.1f MB ffn_share %.2f route_share %.2f' % (d['value'], d['ms_per_step'], r['achieved'], r['ffn_both_phases_gbs'], x['weight_bytes_per_layer']/1e6, x['ffn_ms_share'], x['route_ms_share']))" || tail -5 gpurun_out/sweep.err
done

#!/bin/bash
# is the epilogue the prefill limiter?  DX_GEMM_DBG=8 skips the epilogue math (timing only)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for b in 60 24; do for d in 0 8; do
  echo "== budget $b dbg $d"
  DX_GEMM_DBG=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 --no-batch-sweep --no-q80b --budget-gb $b > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']
print('value %.0f gateup %.0f GB/s | prefill %.0f tok/s %.0f TF/s' % (d['value'], r['achieved'], p['value'], p['gemm_tflops']))" || tail -3 gpurun_out/sweep.err
done; done

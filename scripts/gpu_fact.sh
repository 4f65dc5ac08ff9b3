#!/bin/bash
# factored int decode path: parity tests, then decode bandwidth factored (default) vs exact-dequant (DBG=7)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -5 gpurun_out/gpu_tests.log
for b in 16 24 60; do for d in 0 7; do
  echo "== budget $b dbg $d"
  DX_GEMM_DBG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 --budget-gb $b > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']
print('value %.0f gateup %.0f GB/s both %.0f GB/s | prefill %.0f tok/s %.0f TF/s' % (d['value'], r['achieved'], r['ffn_both_phases_gbs'], p['value'], p['gemm_tflops']))" || tail -3 gpurun_out/sweep.err
done; done

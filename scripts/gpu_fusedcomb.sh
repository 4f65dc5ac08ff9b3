#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -s > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; grep -i "C2 stack\|passed\|failed\|Error" gpurun_out/gpu_tests.log | tail -6
for f in 0 1; do
  echo "== DX_NO_FUSED_COMBINE=$f"
  DX_NO_FUSED_COMBINE=$f timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-batch-sweep > gpurun_out/bench.json 2> gpurun_out/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']
print('value %.0f ms/step %.3f gateup %.0f GB/s | prefill %.0f tok/s %.0f TF/s | e2e %.0f launches %d' % (d['value'], d['ms_per_step'], r['achieved'], p['value'], p['gemm_tflops'], d['e2e']['value'], d['gpu_launches']))" || tail -3 gpurun_out/bench.err
done
